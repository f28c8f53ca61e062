"""Final held-out loss of the reference's teacher-student task over six backward streams (xi salts) for
rtn / sr / sr_fast backward rounding: the spread that tests/test_gpu_teacher.py's hardware-SR tolerance is
based on.  Run from the repo root on a GPU box."""
import os, sys
sys.path.insert(0, os.path.join(os.getcwd(), "tests")); sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2505_14669_b200 as qt
from toy_teacher import Teacher, train
from oracle import oracle as orc
orc.lib()
qt.load()
z = np.load("tests/golden/teacher_runs.npz")
task = Teacher(orc, seed=0)
for s in (0, 1):
    seed = int(z[f"quest_sr_s{s}_seed"])
    for bwd in ("rtn", "sr", "sr_fast"):
        fin = [train(qt, orc, task, seed, fwd="quest", bwd=bwd, xi_salt=k)[1] for k in (None, 1, 2, 3, 4, 5)]
        print(s, bwd, " ".join(f"{f:.5f}" for f in fin), f"mean {np.mean(fin):.5f} sd {np.std(fin):.5f}", flush=True)
