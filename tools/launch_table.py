"""Print per-launch time and DRAM bytes from an `ncu --csv --log-file` launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, data = rows[0], rows[1:]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in data:
    per.setdefault(r[iid], {"k": r[ik].split("(")[0][:60]})[r[im]] = float(r[iv].replace(",", ""))
for i, d in per.items():
    print(f"{i:>4} {d['k']:60s} {d.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us "
          f"{d.get('dram__bytes_read.sum', 0) / 1e6:9.1f} MB rd {d.get('dram__bytes_write.sum', 0) / 1e6:9.1f} MB wr")
