"""Debug: workspace of one 32-bit sort at joint sizes -- digit histograms, coarse joints and the
chunk maps of passes 2-3 against torch recomputations; output vs oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_08929_b200 as B, workloads as W, oracle

def al(x, a=256): return (x + a - 1) // a * a
n = (1 << 24) + 12345
desc = len(sys.argv) > 1 and sys.argv[1] == "desc"
x = W.special_mix(torch.float32, n, 123, "cuda")
s = B.Sorter(torch.float32, n, "cuda")
y = x.clone(); s(y, desc); torch.cuda.synchronize()
ref = oracle.sort_native(x.cpu().numpy(), descending=desc)
got = y.cpu().numpy()
bad = np.flatnonzero(got.view(np.uint32) != ref.view(np.uint32))
print("mismatches", bad.size, bad[:10])
# encoded keys
u = x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
neg = (u >> 31) == 1
enc = torch.where(neg, (~u) & 0xFFFFFFFF, u | 0x80000000)
if desc: enc = (~enc) & 0xFFFFFFFF
ws = s.ws
off = 0
scratch = off; off = al(off + n * 4)
vscr = off; off = al(off + 0)
ghist = off; off = al(off + 4 * 256 * 8 + 16)
bases = off; off = al(off + 4 * 256 * 8)
gcount = off; off = al(off + 4 * 256 * 8)
joint = off
def u64(o, k): return ws[o:o + 8 * k].view(torch.int64).cpu().numpy()
def u32(o, k): return ws[o:o + 4 * k].view(torch.int32).cpu().numpy()
gh = u64(ghist, 1024)
for p in range(4):
    t = torch.bincount(((enc >> (8 * p)) & 255), minlength=256).cpu().numpy()
    print("digit", p, "hist ok", np.array_equal(gh[p*256:(p+1)*256], t))
gc_off = joint + 65536 * 8
gco = u64(gc_off, 2048)
c2 = torch.bincount(((enc >> 14) & 3) * 256 + ((enc >> 16) & 255), minlength=1024).cpu().numpy()
c3 = torch.bincount(((enc >> 22) & 3) * 256 + ((enc >> 24) & 255), minlength=1024).cpu().numpy()
print("coarse2 ok", np.array_equal(gco[:1024], c2), "coarse3 ok", np.array_equal(gco[1024:], c3))
cs_off = gc_off + 2048 * 8
cs = u64(cs_off, 10); ct = u32(cs_off + 80, 10); jp = u32(cs_off + 80 + 40, 2048)
print("cstart", cs); print("ctile", ct)
bs = u64(bases, 1024)
for q in range(2):
    p = 2 + q
    cc = (c2 if q == 0 else c3).reshape(4, 256)
    exp = bs[p*256:(p+1)*256][None, :] + np.concatenate([np.zeros((1, 256), np.int64), np.cumsum(cc, 0)[:-1]])
    print("jp", p, "ok", np.array_equal(jp[q*1024:(q+1)*1024].reshape(4, 256), exp))
t2 = torch.bincount(((enc >> 16) & 255), minlength=256).cpu().numpy()
print("d2 got", gh[512:520], "sum", gh[512:768].sum())
print("d2 exp", t2[:8], "sum", t2.sum())
print("coarse2 col sums", c2.reshape(4, 256).sum(0)[:8])
print("d3 got sum", gh[768:1024].sum(), "exp", n)
