"""Summarise an ncu --csv launch list (gpu__time_duration, dram bytes) of libbsort's kernels:
one line per launch of a k_* kernel, plus GB/s of algorithmic vs measured traffic."""
import csv
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = {}
    for r in rows[1:]:
        d.setdefault(int(r[ii]), {"kernel": r[ki]})[r[mi]] = r[vi]
    return [d[k] for k in sorted(d) if "k_" in d[k]["kernel"]]


if __name__ == "__main__":
    for path in sys.argv[1:]:
        print(path)
        for v in launches(path):
            ns = float(v.get("gpu__time_duration.sum", "nan"))
            rd = float(v.get("dram__bytes_read.sum", "0"))
            wr = float(v.get("dram__bytes_write.sum", "0"))
            name = v["kernel"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:70]
            extra = {k: v[k] for k in v if k not in ("kernel", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                                      "dram__bytes_write.sum")}
            print(f"  {ns / 1e3:9.1f} us  dram {rd / 1e6:9.1f} MB rd {wr / 1e6:9.1f} MB wr  "
                  f"{(rd + wr) / ns if ns else 0:7.1f} GB/s  {name} {extra if extra else ''}")
