"""Per-opcode shared-memory wavefronts (actual vs ideal) and executed instructions from an ncu report."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout)))
h = src[1]; data = src[2:]
iw, ii, ie = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal"), h.index("Instructions Executed")
agg = collections.defaultdict(lambda: [0, 0, 0])
tot_inst = 0
for r in data:
    op = r[1].split()
    if not op: continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0] + ("." + o.split(".")[1] if o.startswith(("LDS", "STS", "ATOMS")) and "." in o else "")
    try:
        w, i, e = int(r[iw] or 0), int(r[ii] or 0), int(r[ie] or 0)
    except ValueError:
        continue
    agg[o][0] += w; agg[o][1] += i; agg[o][2] += e
    tot_inst += e
keys = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 30
print(f"total warp-instructions {tot_inst}  per 32 keys {tot_inst / (keys / 32):.2f}")
tw = sum(v[0] for v in agg.values())
print(f"total smem wavefronts {tw}  per 32 keys {tw / (keys / 32):.2f}")
for o, (w, i, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:12]:
    if w: print(f"  {o:12s} wavefronts/32keys {w/(keys/32):6.2f}  ideal {i/(keys/32):6.2f}  instr/32keys {e/(keys/32):6.2f}")
print("top opcodes by count:")
for o, (w, i, e) in sorted(agg.items(), key=lambda x: -x[1][2])[:25]:
    print(f"  {o:14s} {e/(keys/32):6.2f}")
