"""Per-source-line executed warp instructions of an ncu report (needs -lineinfo)."""
import csv
import io
import subprocess
import sys


def main(rep, top=40, keys=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, res = None, None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or not r[0]:
            continue
        try:
            ie = int(r[hdr.index("Instructions Executed")])
        except ValueError:
            continue
        res.append((ie, fname, r[0], r[1][:100]))
    tot = sum(x[0] for x in res)
    print(f"total warp instructions {tot:.4g}" + (f"  = {tot * 32 / keys:.1f} per 32 keys" if keys else ""))
    for ie, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
        extra = f" {ie * 32 / keys:6.2f}/32k" if keys else ""
        print(f"{100*ie/tot:5.1f}%{extra} {f}:{ln:5s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, float(sys.argv[3]) if len(sys.argv) > 3 else None)
