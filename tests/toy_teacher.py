"""Test harness: the reference's toy training loop (mx4train/train.py) restated, with every quantized
linear layer executed by the B200 path (paper_2505_14669_b200.forward / backward -> libquartet_b200).

Only the layer calls change; data, initialisation, the ReLU MLP, the loss and AdamW follow the
reference line by line (test infrastructure -- the toy harness itself is out of scope as a product):
  ToyModel init                 train.py:91-106  (rng.gaussians(derive_seed(seed, 1, layer)) * sqrt(2/d_in))
  TeacherStudentTask            train.py:182-227 (teacher 64 -> 512 -> 32, label noise 0.5)
  model_forward / backward      train.py:131-159 (ReLU between layers, xi = derive_seed(xi_step, layer))
  train loop + AdamW            train.py:325-382 (lr_at, global-norm clip 1.0, bias-corrected AdamW)
  evaluate                      train.py:384-393 (held-out batch of 2048, forward seed derive_seed(task, 3))
"""

from __future__ import annotations

import math

import numpy as np
import torch

T_INIT, T_DATA, T_EVAL, T_XI, T_SRFWD, T_TEACHER = 1, 2, 3, 4, 5, 6
DIMS = [64, 128, 128, 64, 32]


class Teacher:
    def __init__(self, orc, seed=0, d_in=64, d_out=32, hidden=512, noise=0.5):
        self.o, self.seed, self.d_in, self.noise = orc, seed, d_in, noise
        g = orc.DOMAIN_GAUSS
        w1 = orc.gaussians(orc.derive_seed(seed, T_TEACHER, 1), g, 0, hidden * d_in)
        w2 = orc.gaussians(orc.derive_seed(seed, T_TEACHER, 2), g, 0, d_out * hidden)
        self.w1 = (w1.reshape(hidden, d_in) * math.sqrt(2.0 / d_in)).astype(np.float32)
        self.w2 = (w2.reshape(d_out, hidden) * math.sqrt(1.0 / hidden)).astype(np.float32)

    def _targets(self, x, noise_seed):
        t = np.maximum(x @ self.w1.T, 0.0) @ self.w2.T
        eps = self.o.gaussians(noise_seed, self.o.DOMAIN_GAUSS, 0, t.size).reshape(t.shape)
        return t + self.noise * eps.astype(np.float32)

    def batch(self, seed, step, n):
        o = self.o
        x = o.gaussians(o.derive_seed(seed, T_DATA, step), o.DOMAIN_GAUSS, 0, n * self.d_in)
        x = x.reshape(n, self.d_in).astype(np.float32)
        return x, self._targets(x, o.derive_seed(seed, T_DATA, step, 1))

    def eval_batch(self, n):
        o = self.o
        x = o.gaussians(o.derive_seed(self.seed, T_EVAL), o.DOMAIN_GAUSS, 0, n * self.d_in)
        x = x.reshape(n, self.d_in).astype(np.float32)
        return x, self._targets(x, o.derive_seed(self.seed, T_EVAL, 1))

    @staticmethod
    def loss_grad(y, target):
        diff = (y - target).astype(np.float64)
        return float((diff * diff).mean()), (2.0 * diff / diff.size).astype(np.float32)


def init_weights(orc, seed):
    ws = []
    for layer, (di, do) in enumerate(zip(DIMS[:-1], DIMS[1:])):
        w = orc.gaussians(orc.derive_seed(seed, T_INIT, layer), orc.DOMAIN_GAUSS, 0, do * di)
        ws.append((w.reshape(do, di) * math.sqrt(2.0 / di)).astype(np.float32))
    return ws


def lr_at(step, steps=400, lr=0.02, warmup_frac=0.1, lr_floor=0.0):
    warmup = max(1, int(round(warmup_frac * steps)))
    if step < warmup:
        return lr * (step + 1) / warmup
    span = max(1, steps - 1 - warmup)
    t = min(step - warmup, span)
    return lr_floor + 0.5 * (lr - lr_floor) * (1.0 + math.cos(math.pi * t / span))


def _fwd(qt, x, w, fwd, seed, layer, step):
    scheme = {"quest": qt.QUEST, "rtn": qt.RTN_ABSMAX, "sr": qt.SR_ABSMAX}[fwd]
    sr_seed = qt.derive_seed(seed, T_SRFWD, step, layer) if fwd == "sr" else None
    y, ctx = qt.forward(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), scheme=scheme, seed=sr_seed)
    return y.cpu().numpy(), ctx


def model_forward(qt, ws, x, fwd, seed, step):
    a, acts, caches = np.asarray(x, np.float32), [np.asarray(x, np.float32)], []
    for layer, w in enumerate(ws):
        z, ctx = _fwd(qt, a, w, fwd, seed, layer, step)
        caches.append(ctx)
        a = np.maximum(z, 0.0) if layer < len(ws) - 1 else z
        acts.append(a)
    return acts, caches


def model_backward(qt, ws, acts, caches, dy, bwd, xi):
    grads = [None] * len(ws)
    g = np.asarray(dy, np.float32)
    for layer in range(len(ws) - 1, -1, -1):
        if layer < len(ws) - 1:
            g = g * (acts[layer + 1] > 0.0)
        dx, dw = qt.backward(torch.from_numpy(np.ascontiguousarray(g)).cuda(), caches[layer],
                             xi=qt.derive_seed(xi, layer), rounding=bwd)
        grads[layer] = dw.cpu().numpy()
        g = dx.cpu().numpy()
    return grads


def train(qt, orc, task, seed, fwd="quest", bwd="rtn", steps=400, batch=64, lr=0.02, wd=0.1, clip=1.0,
          b1=0.9, b2=0.95, eps=1e-8, eval_every=10, xi_salt=None):
    ws = init_weights(orc, seed)
    ms = [np.zeros_like(w) for w in ws]
    vs = [np.zeros_like(w) for w in ws]
    history = []
    for step in range(steps):
        lr_s = lr_at(step, steps, lr)
        x, target = task.batch(seed, step, batch)
        acts, caches = model_forward(qt, ws, x, fwd, seed, step)
        loss, dy = task.loss_grad(acts[-1], target)
        if step % eval_every == 0 or step == steps - 1:
            history.append((step, loss, lr_s))
        xi = qt.derive_seed(seed, T_XI, step) if xi_salt is None else qt.derive_seed(seed, T_XI, step, xi_salt)
        grads = model_backward(qt, ws, acts, caches, dy, bwd, xi)   # xi_salt: other backward streams (tests)
        gnorm = math.sqrt(sum(float(np.sum(g.astype(np.float64) ** 2)) for g in grads))
        if gnorm > clip:
            sc = np.float32(clip / gnorm)
            grads = [g * sc for g in grads]
        t = step + 1
        bc1, bc2 = 1.0 - b1 ** t, 1.0 - b2 ** t
        for w, g, m, v in zip(ws, grads, ms, vs):
            m *= b1
            m += (1.0 - b1) * g
            v *= b2
            v += (1.0 - b2) * g * g
            w *= 1.0 - lr_s * wd
            w -= (lr_s / bc1) * m / (np.sqrt(v / bc2) + eps)
    x, target = task.eval_batch(2048)
    acts, _ = model_forward(qt, ws, x, fwd, orc.derive_seed(task.seed, T_EVAL), 0)
    final = task.loss_grad(acts[-1], target)[0]
    history.append((steps, final, lr_at(steps - 1, steps, lr)))
    return np.array(history), final
