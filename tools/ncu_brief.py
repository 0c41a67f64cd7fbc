"""Brief of an ncu --set full report: SOL, occupancy, top stall reasons, per kernel."""
import csv
import io
import subprocess
import sys


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1])) if len(rows) > 1 else {}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        name = d.get("Kernel Name", "?")[:40]
        def g(k):
            try:
                return float(d.get(k, "nan").replace(",", ""))
            except ValueError:
                return float("nan")
        tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(
            units.get("gpu__time_duration.sum", "ns"), 1e-3)
        def bsc(k):  # read and write sums can come in different units
            return {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(units.get(k, "byte"), 1e-9)
        print(f"== {name}  dur {g('gpu__time_duration.sum')*tscale:.1f} us  dram {g('dram__throughput.avg.pct_of_peak_sustained_elapsed'):.1f}%  "
              f"sm {g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f}%  occ {g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}%  "
              f"regs {g('launch__registers_per_thread'):.0f}  L2hit {g('lts__t_sector_hit_rate.pct'):.1f}%  "
              f"dramGB {g('dram__bytes_read.sum')*bsc('dram__bytes_read.sum')+g('dram__bytes_write.sum')*bsc('dram__bytes_write.sum'):.3f}")
        st = [(k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), g(k))
              for k in hdr if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
        st = sorted([s for s in st if s[1] == s[1]], key=lambda s: -s[1])[:6]
        print("   stalls: " + ", ".join(f"{k} {v:.2f}" for k, v in st))
        pipes = [(k.replace('sm__inst_executed_pipe_', '').replace('.avg.pct_of_peak_sustained_active', ''), g(k))
                 for k in hdr if k.startswith('sm__inst_executed_pipe_') and k.endswith('.avg.pct_of_peak_sustained_active')]
        pipes = sorted([p for p in pipes if p[1] == p[1] and p[1] > 5], key=lambda p: -p[1])[:6]
        print("   pipes: " + ", ".join(f"{k} {v:.1f}%" for k, v in pipes))


if __name__ == "__main__":
    for r in sys.argv[1:]:
        main(r)
