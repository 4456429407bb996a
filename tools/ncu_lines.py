"""Per-source-line stall samples of an ncu report (needs -lineinfo): top lines with stall mix."""
import csv
import io
import subprocess
import sys


def main(rep, top=40):
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
        if hdr is None or len(r) < 5 or not r[0]:
            continue
        iS = 4
        try:
            s = int(r[iS])
        except ValueError:
            continue
        stalls = {hdr[i]: r[i] for i in range(len(hdr)) if hdr[i].startswith("stall_") and r[i] not in ("0", "", "-")}
        res.append((s, fname, r[0], r[1][:90], stalls))
    tot = sum(x[0] for x in res)
    for s, f, ln, src, st in sorted(res, key=lambda x: -x[0])[:top]:
        det = " ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda kv: -int(kv[1]) if kv[1].isdigit() else 0)[:4])
        print(f"{100*s/tot:5.1f}% {f}:{ln:5s} {src:90s} {det}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
