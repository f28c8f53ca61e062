"""The bench's end-to-end pipeline (upload / compute / download streams, double-buffered device inputs,
Johnson shape order) downloads exactly what the serial public-API calls produce."""

import pytest
import torch


def test_johnson_order_cpu_rule():
    import bench

    # upload-light / download-heavy jobs first by increasing upload, then the rest by decreasing download
    assert bench.johnson_order([268, 495, 495], [201, 314, 540]) == [2, 1, 0]
    assert bench.johnson_order([1, 5, 3], [4, 2, 6]) == [0, 2, 1]


@pytest.mark.gpu
def test_e2e_pipeline_matches_serial_calls():
    import bench
    import paper_2505_14669_b200 as qt

    qt.load()
    g = torch.Generator(device="cuda").manual_seed(5)
    T = 512
    data = []
    for d_in, d_out in [(256, 256), (256, 512), (512, 256)]:
        x = torch.randn(T, d_in, device="cuda", generator=g).to(torch.bfloat16)
        w = torch.randn(d_out, d_in, device="cuda", generator=g) / d_in ** 0.5
        dy = torch.randn(T, d_out, device="cuda", generator=g).to(torch.bfloat16)
        data.append((x, w, dy))
    steps = 3
    outs = []
    res = bench.e2e_pipeline(qt, data, torch.device("cuda"), steps, outs_sink=outs)
    assert res["h2d_bytes_per_step"] == sum(x.numel() * 2 + dy.numel() * 2 for x, _, dy in data)
    xi = 100 + steps - 1
    for i, ((x, w, dy), (ox, ow)) in enumerate(zip(data, outs)):
        _, ctx = qt.forward(x, w, out_dtype=torch.bfloat16, check_finite=False, bwd_xi=xi * 3 + i)
        dx, dw = qt.backward(dy, ctx, xi=xi * 3 + i, dx_dtype=torch.bfloat16, check_finite=False)
        assert torch.equal(ox, dx.cpu()), i
        assert torch.equal(ow, dw.cpu()), i
