import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2603_08929_b200 as B, workloads as W
n = int(sys.argv[1]); dt = getattr(torch, sys.argv[2]); mode = sys.argv[3]
x = W.special_mix(dt, n, 123, "cuda") if dt.is_floating_point else W.uniform_int(dt, n, 123, "cuda")
if mode == "inelig":
    ib = {4: torch.int32, 8: torch.int64}[x.element_size()]
    b = x.view(ib).clone(); low = b & 0xFF
    b = torch.where(low == 0x42, b + 1, b); b[:100] = (b[:100] & ~0xFF) | 0x42; x = b.view(dt)
torch.cuda.synchronize(); t0 = time.time()
B.sort_(x); torch.cuda.synchronize()
print("ok", n, dt, mode, time.time() - t0, flush=True)
