"""2 ranks on one GPU (gloo): LU b=256 with keep_input/reset (bench path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("gloo")
import paper_2301_03166_b200 as P
from paper_2301_03166_b200.distributed import DistributedFactorization
n, b = int(sys.argv[1]), int(sys.argv[2])
a = P.generate_test_matrix("lu", n, 0)
for keep in (False, True):
    f = DistributedFactorization("lu", a, b, keep_input=keep)
    if keep:
        f.reset()
    try:
        reps = f.run_protected("full", {}, np.random.default_rng(0))
        print(dist.get_rank(), "keep", keep, "ok", f.residual(a), flush=True)
    except Exception as e:
        print(dist.get_rank(), "keep", keep, "FAIL", e, flush=True)
    del f
dist.destroy_process_group()
