"""Time / profile the diagonal-block factorization kernels on device pointers:
python tools/prof/diag_probe.py [variant] [mode] [w] [reps]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2301_03166_b200 import _lib

variant, mode, w, reps = (int(x) for x in (sys.argv[1:] + ["1", "0", "256", "20"][len(sys.argv) - 1:]))
lib = _lib.load()
rng = np.random.default_rng(0)
a = rng.uniform(-1, 1, (w, w))
a = a @ a.T + w * np.eye(w) if mode == 1 else a + np.diag(np.abs(a).sum(1) + 1)
src = torch.from_numpy(a.T.copy()).cuda()
D = src.clone()
Li = torch.zeros_like(D)
Ui = torch.zeros_like(D)
sg = torch.zeros(w, dtype=torch.float64, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for i in range(reps):
    D.copy_(src)
    torch.cuda.synchronize()
    ev[0].record()
    lib.abft_dev_diag_factor(None, variant, mode, w, D.data_ptr(), w, Li.data_ptr(), w,
                             Ui.data_ptr() if mode != 1 else None, w, info.data_ptr(), sg.data_ptr())
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
print(f"variant {variant} mode {mode} w {w}: median {np.median(ts[2:]):.1f} us (min {min(ts):.1f})")
