"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys


def main(rep, top=25, kernel_idx=0):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = raw.split('"Kernel Name"')
    blk = blocks[kernel_idx + 1] if len(blocks) > kernel_idx + 1 else blocks[-1]
    rows = list(csv.reader(io.StringIO('"Kernel Name"' + blk)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = []
    total = 0
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        try:
            smp = int(r[idx["Warp Stall Sampling (All Samples)"]])
        except ValueError:
            continue
        total += smp
        stalls = {h: r[i] for h, i in idx.items() if h.startswith("stall_") and "Not Issued" not in h}
        top_st = sorted(((int(v), k) for k, v in stalls.items() if v.isdigit() and int(v) > 0), reverse=True)[:3]
        data.append((smp, r[idx["Address"]][-5:], r[idx["Source"]].strip()[:60], top_st))
    data.sort(reverse=True)
    print(f"{rows[0][1][:60]}  total samples {total}")
    for smp, a, src, st in data[:top]:
        print(f"{smp:7d} {100.0 * smp / max(1, total):5.1f}% {a} {src:60s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25,
         int(sys.argv[3]) if len(sys.argv) > 3 else 0)
