"""Summarise an ncu --csv launch list: per kernel name -> launches, mean us, GB moved, GB/s."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hdr_i]
    out = defaultdict(dict)
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        try:
            out[key][d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
        except ValueError:
            pass
    return out


def traffic(path):
    """{kernel short name: mean DRAM bytes (read + write) per launch}."""
    data = load(path)
    agg = defaultdict(lambda: [0, 0.0])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for (i, name), m in data.items():
        short = name.split("(")[0].replace("void ", "").replace("dagrt::", "").split("<")[0]
        if "dram__bytes_read.sum" not in m:
            continue
        b = sum(m[k][0] * scale.get(m[k][1], 0) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
        agg[short][0] += 1
        agg[short][1] += b
    return {k: v[1] / v[0] for k, v in agg.items() if v[0]}


def main(path, peak=6540.8):
    data = load(path)
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
    for (i, name), m in data.items():
        short = name.split("(")[0].replace("void ", "").replace("dagrt::", "")
        t = m.get("gpu__time_duration.sum", (0, ""))
        tus = t[0] * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                      "msecond": 1e3}.get(t[1], 1.0)
        rd = m.get("dram__bytes_read.sum", (0, ""))
        wr = m.get("dram__bytes_write.sum", (0, ""))
        def gb(x):
            v, u = x
            return v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "B": 1e-9,
                        "KB": 1e-6, "MB": 1e-3, "GB": 1.0}.get(u, 0)
        a = agg[short]
        a[0] += 1; a[1] += tus; a[2] += gb(rd) + gb(wr)
        a[3] += m.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", (0, ""))[0]
        a[4] += m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed", (0, ""))[0]
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':28s} {'n':>4s} {'mean_us':>9s} {'share':>6s} {'GB/launch':>10s} {'GB/s':>8s} {'%peak':>6s} {'sm%':>5s} {'dram%':>6s}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        n, t, g = a[0], a[1], a[2]
        bw = g / (t * 1e-6) if t else 0
        print(f"{k[:28]:28s} {n:4d} {t / n:9.1f} {t / tot:6.1%} {g / n:10.4f} {bw:8.0f} {bw / peak:6.1%} {a[3] / n:5.1f} {a[4] / n:6.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
