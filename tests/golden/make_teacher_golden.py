"""Golden loss histories of the reference's own toy training loop (teacher-student task), for the
end-to-end loss-parity test tests/test_gpu_teacher.py.

    python tests/golden/make_teacher_golden.py      (build container only; imports /root/reference)

Runs mx4train.train.train (train.py:325-382) on make_task("teacher", seed=0) with the selftest's run
seeds (selftest.py:_training_runs: derive_seed(0, 11, s) & 0xFFFFFFFF) for the quest:rtn and quest:sr
pairs and records the loss history (every eval_every = 10 steps) and the final held-out loss.
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import HERE, _import_reference  # noqa: E402


def main():
    mx = _import_reference()
    from mx4train import rng, train

    task = train.make_task("teacher", seed=0)
    out = {}
    for label in ("quest:rtn", "quest:sr"):
        fwd, bwd = label.split(":")
        for s in range(2):
            run_seed = rng.derive_seed(0, 11, s) & 0xFFFFFFFF
            cfg = train.TrainConfig(seed=run_seed)
            model = train.ToyModel(train.DEFAULT_DIMS["teacher"], seed=run_seed, pair=train.SchemePair(fwd, bwd))
            r = train.train(model, task, cfg)
            key = f"{fwd}_{bwd}_s{s}"
            out[f"{key}_history"] = np.array([[st, lo, lr] for st, lo, lr in r.history], np.float64)
            out[f"{key}_final"] = np.float64(r.final_loss)
            out[f"{key}_seed"] = np.uint64(run_seed)
            print(key, r.status, r.final_loss)
    np.savez_compressed(os.path.join(HERE, "teacher_runs.npz"), **out)


if __name__ == "__main__":
    main()
