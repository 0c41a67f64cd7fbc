"""Markdown tables of one default bench.py line (the six-benchmark suite):
    python tools/suite_table.py gpurun_out/jNN/bench.json >> profiles/rN_summary.md"""
import json
import sys


def rows(d):
    yield d["config"]["bench"], d
    for k, v in d.get("suite", {}).items():
        yield k, v


def main(path):
    d = json.loads(open(path).read().strip().splitlines()[-1])
    f = lambda x, n=3: "-" if x is None else f"{x:.{n}f}"  # noqa: E731
    print("## bench.py suite (ms per DAG; resident = inputs in HBM; e2e = stream mode, H2D/D2H inside)\n")
    print("| bench | dagrt resident | serial | CUDA graph | f1 cache | single-stream | e2e (stream) | serial | "
          "CUDA graph | prefetch off | UM prefetch | UM faults | UM serial faults | R_cp frac | R_work frac | "
          "Fig. 9 est. | kernel | roofline frac |")
    print("|" + "---|" * 19)
    for name, r in rows(d):
        b = r.get("baselines", {})
        dr = r.get("dag_roofline", {})
        cf = r.get("contention_free", {})
        rf = r.get("roofline", {})
        print(f"| {name} | {f(r['value'])} | {f(b.get('serial_resident_ms'))} | {f(b.get('graph_resident_ms'))} | "
              f"{f(b.get('f1_graph_cache_resident_ms'))} | {f(b.get('single_stream_resident_ms'))} | "
              f"{f(r['e2e']['value'])} | {f(b.get('serial_stream_ms'))} | {f(b.get('graph_stream_ms'))} | "
              f"{f(b.get('parallel_no_prefetch_stream_ms'))} | {f(b.get('um_parallel_prefetch_ms'), 1)} | "
              f"{f(b.get('um_parallel_fault_ms'), 1)} | {f(b.get('um_serial_fault_ms'), 1)} | "
              f"{f(dr.get('frac_cp'))} | {f(dr.get('frac_work'))} | {f(cf.get('resident_ms'))} | "
              f"{rf.get('kernel')} | {f(rf.get('frac'))} |")
    g = d.get("suite_geomean", {})
    print("\nGeomeans over the six: " + ", ".join(f"{k} {v:.3f}" for k, v in g.items() if isinstance(v, float)))
    sch = d.get("scheduler", {})
    if sch:
        print(f"\nHost cost per launch (B&S DAG): {sch.get('sched_us_per_launch'):.2f} us = "
              + ", ".join(f"{k} {v:.2f}" for k, v in sch.get("breakdown_us_per_launch", {}).items()))
    print(f"\nClocks: {json.dumps(d.get('clocks'))}\n")
    print("Per-kernel rooflines (each kernel alone, serial-sync region, event-timed):\n")
    print("| bench | kernel | launches/DAG | avg us | algorithmic MB | GB/s | HBM frac | share of serial DAG |")
    print("|---|---|---|---|---|---|---|---|")
    for name, r in rows(d):
        for k in r.get("kernel_rooflines") or []:
            print(f"| {name} | {k['kernel']} | {k['launches_per_dag']} | {1e3 * k['avg_launch_ms']:.1f} | "
                  f"{k['algorithmic_bytes_per_launch'] / 1e6:.1f} | {f(k['achieved_gbs'], 0)} | {f(k['hbm_frac'])} | "
                  f"{f(k['share_of_serial_dag'])} |")
    print()


if __name__ == "__main__":
    main(sys.argv[1])
