"""Summarise an ncu report: key SOL metrics, pipe utilisation, top stall sites (SASS)."""
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, top=30):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u = raw[0], raw[1]
    for row in raw[2:]:
        print("kernel:", row[h.index("Kernel Name")][:140])
        want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum"]
        for w in want:
            if w in h:
                print(f"  {w} = {row[h.index(w)]} {u[h.index(w)]}")
        for i, name in enumerate(h):
            if name.startswith("sm__inst_executed_pipe_") and name.endswith("avg.pct_of_peak_sustained_active"):
                try:
                    if float(row[i]) > 5:
                        print(f"  {name} = {row[i]}")
                except ValueError:
                    pass
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hh = src[1]
    data = src[2:]
    iS = hh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
    stalls = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
    agg = {c: sum(int(r[hh.index(c)]) for r in data if r[hh.index(c)].isdigit()) for c in stalls}
    print("stall totals (% of samples):", ", ".join(f"{k[6:]}={100*v/tot:.1f}" for k, v in
                                                    sorted(agg.items(), key=lambda x: -x[1]) if v > tot * 0.01))
    print("top instructions:")
    for r in sorted(data, key=lambda r: -int(r[iS]) if r[iS].isdigit() else 0)[:top]:
        det = " ".join(f"{c[6:]}={r[hh.index(c)]}" for c in stalls if r[hh.index(c)] not in ("0", ""))
        print(f"  {int(r[iS])*100/tot:5.1f}%  {r[1][:58]:58s} {det}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
