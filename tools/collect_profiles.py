"""Summarise a GPU round (gpurun_out/) into profiles/<tag>_*.md / .csv.

    python tools/collect_profiles.py r1
"""
import glob
import io
import json
import os
import shutil
import subprocess
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def main(tag, src=None):
    global OUT
    if src:
        OUT = os.path.abspath(src)
    import ncu_summary
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# GPU round {tag}: benchmarks, ncu launch lists, schedule overlap\n"]
    lines.append("## bench.py lines (ms per DAG; resident = inputs in HBM; stream = e2e with H2D/D2H)\n")
    lines.append("| bench | dagrt resident | serial | CUDA graph | f1 cache | dagrt stream (e2e) | serial | CUDA graph | f1 cache | roofline kernel | frac | clocks |")
    lines.append("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for b in ["vec", "bs", "img", "ml", "hits", "dl"]:
        p = os.path.join(OUT, f"bench_{b}.json")
        if not os.path.exists(p):
            continue
        try:
            d = json.load(open(p))
        except Exception:
            continue
        bl = d.get("baselines", {})
        r = d["roofline"]
        f = lambda k: f"{bl[k]:.3f}" if k in bl else "-"
        lines.append(f"| {b} | {d['value']:.3f} | {f('serial_resident_ms')} | {f('graph_resident_ms')} | "
                     f"{f('f1_graph_cache_resident_ms')} | {d['e2e']['value']:.3f} | {f('serial_stream_ms')} | "
                     f"{f('graph_stream_ms')} | {f('f1_graph_cache_stream_ms')} | {r['kernel']} | "
                     f"{(r['frac'] or 0):.3f} | {d['clocks'].get('sm_mhz')} MHz {d['clocks'].get('reasons')} |")
        shutil.copy(p, os.path.join(PROF, f"{tag}_bench_{b}.json"))
    lines.append("")
    abl = []
    for b in ["vec", "bs", "img", "ml", "hits", "dl"]:
        p = os.path.join(OUT, f"bench_{b}.json")
        try:
            d = json.load(open(p))
        except Exception:
            continue
        bl = d.get("baselines", {})
        if "parallel_no_prefetch_stream_ms" in bl:
            abl.append(f"| {b} | {d['e2e']['value']:.3f} | {bl['parallel_no_prefetch_stream_ms']:.3f} | "
                       f"{bl.get('serial_stream_ms', float('nan')):.3f} |")
    if abl:
        lines.append("## Ablation: the prefetcher (stream mode, ms per DAG; PAPER.md L356-366)\n")
        lines.append("| bench | parallel + prefetch | parallel, prefetch off | serial-sync |")
        lines.append("|---|---|---|---|")
        lines += abl
        lines.append("")
    traffic = {}
    for csvp in sorted(glob.glob(os.path.join(OUT, "ncu_*.csv"))):
        b = os.path.basename(csvp)[4:-4]
        buf = io.StringIO()
        with redirect_stdout(buf):
            ncu_summary.main(csvp)
        lines.append(f"## ncu launch list: {b} (2 DAG runs, serialised, cold-ish cache)\n")
        lines.append("```")
        lines.append(buf.getvalue().rstrip())
        lines.append("```\n")
        shutil.copy(csvp, os.path.join(PROF, f"{tag}_ncu_{b}.csv"))
        traffic[b] = ncu_summary.traffic(csvp)
    ov = sorted(glob.glob(os.path.join(OUT, "overlap_*.json")))
    if ov:
        lines.append("## Schedule overlap (PAPER.md §V-F metrics, from the scheduler's event timeline)\n")
        lines.append("| bench | mode | policy | CT | TC | CC | TOT | span ms/DAG |")
        lines.append("|---|---|---|---|---|---|---|---|")
        for p in ov:
            d = json.load(open(p))
            for pol in ("parallel", "serial"):
                m = d.get(pol)
                if m:
                    lines.append(f"| {d['bench']} | {d['mode']} | {pol} | {m['CT']:.2f} | {m['TC']:.2f} | "
                                 f"{m['CC']:.2f} | {m['TOT']:.2f} | {m['span_ms']:.3f} |")
            shutil.copy(p, os.path.join(PROF, f"{tag}_{os.path.basename(p)}"))
        lines.append("")
    ovk = sorted(glob.glob(os.path.join(OUT, "ovk_*.json")))
    if ovk:
        lines.append("## Schedule overlap from a CUPTI (kineto) trace (PAPER.md §V-F L1272-1283)\n")
        lines.append("| bench | mode | policy | CT | TC | CC | TOT | span ms/DAG |")
        lines.append("|---|---|---|---|---|---|---|---|")
        for p in ovk:
            d = json.load(open(p))
            for pol in ("parallel", "serial"):
                m = d.get(pol)
                if m:
                    lines.append(f"| {d.get('bench')} | {d.get('mode')} | {pol} | {m['CT']:.2f} | {m['TC']:.2f} | "
                                 f"{m['CC']:.2f} | {m['TOT']:.2f} | {m.get('span_ms', float('nan')):.3f} |")
            shutil.copy(p, os.path.join(PROF, f"{tag}_{os.path.basename(p)}"))
        lines.append("")
    san = sorted(glob.glob(os.path.join(OUT, "sanitize_*.log")))
    if san:
        lines.append("## compute-sanitizer (small parity tests of every benchmark)\n")
        lines.append("```")
        for p in san:
            tail = [l for l in open(p).read().splitlines() if "SUMMARY" in l or "passed" in l or l.startswith("rc=")]
            lines.append(f"{os.path.basename(p)}: " + " | ".join(tail))
            shutil.copy(p, os.path.join(PROF, f"{tag}_{os.path.basename(p)}"))
        lines.append("```\n")
    for rep in sorted(glob.glob(os.path.join(OUT, "prof_*.ncu-rep"))):
        import ncu_brief
        buf = io.StringIO()
        with redirect_stdout(buf):
            ncu_brief.main(rep)
        lines.append(f"## ncu --set full: {os.path.basename(rep)}\n")
        lines.append("```")
        lines.append(buf.getvalue().rstrip())
        lines.append("```\n")
    if traffic:  # read by bench.py for roofline.traffic (DRAM bytes per launch, ncu)
        with open(os.path.join(PROF, f"{tag}_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1, sort_keys=True)
    # the default bench line, the reference arm, the B&S FP64 op count, the GPU test result
    extra = [("bench_default.json", "bench_default.json"), ("bench_reference.json", "bench_reference.json"),
             ("fp64_bs.csv", "fp64_bs.csv"), ("smoke.log", "smoke.log")]
    for src, dst in extra:
        sp = os.path.join(OUT, src)
        if os.path.exists(sp):
            shutil.copy(sp, os.path.join(PROF, f"{tag}_{dst}"))
    pl = os.path.join(OUT, "pytest_gpu.log")
    if os.path.exists(pl):
        tail = open(pl).read().strip().splitlines()[-3:]
        with open(os.path.join(PROF, f"{tag}_pytest_gpu.txt"), "w") as f:
            f.write("\n".join(tail) + "\n")
        lines.append("## pytest -m gpu\n")
        lines.append("```")
        lines.extend(tail)
        lines.append("```\n")
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1", sys.argv[2] if len(sys.argv) > 2 else None)
