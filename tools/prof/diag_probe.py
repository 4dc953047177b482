"""Time the diagonal-block factorization kernels on device pointers:
python tools/prof/diag_probe.py [variant] [mode] [w] [reps] [f64|f32]
variant (abft_dev_diag_factor): 0 unblocked one-CTA, 1 blocked multi-CTA
(cooperative). ABFT_LIB=<path> times another build of the library (A/B).
`reps` launches run back to back on
distinct copies of the block (steady clocks, no host sync in between); the
mean per launch is printed."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2301_03166_b200 import _lib

args = sys.argv[1:5] + ["1", "0", "256", "50"][len(sys.argv[1:5]):]
variant, mode, w, reps = (int(x) for x in args)
prec = sys.argv[5] if len(sys.argv) > 5 else "f64"
lib = _lib.load()
rng = np.random.default_rng(0)
a = rng.uniform(-1, 1, (w, w))
a = a @ a.T + w * np.eye(w) if mode == 1 else a + np.diag(np.abs(a).sum(1) + 1)
if mode == 2:
    a = np.linalg.qr(rng.standard_normal((w, w)))[0]
dt = torch.float64 if prec == "f64" else torch.float32
fn = lib.abft_dev_diag_factor if prec == "f64" else lib.abft_dev_sdiag_factor
src = torch.from_numpy(a.T.copy()).to(dt).cuda()
D = src.unsqueeze(0).repeat(reps + 5, 1, 1).contiguous()
Li = torch.zeros_like(D)
Ui = torch.zeros_like(D)
sg = torch.zeros(w, dtype=dt, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")


def launch(i):
    rc = fn(None, variant, mode, w, D[i].data_ptr(), w, Li[i].data_ptr(), w,
            Ui[i].data_ptr() if mode != 1 else None, w, info.data_ptr(), sg.data_ptr())
    assert rc == 0, _lib.last_error()


for i in range(5):
    launch(i)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for i in range(5, reps + 5):
    launch(i)
ev[1].record()
torch.cuda.synchronize()
us = ev[0].elapsed_time(ev[1]) * 1e3 / reps
print(f"{prec} variant {variant} mode {mode} w {w}: info {int(info.item())} mean {us:.1f} us over {reps} back-to-back launches")
