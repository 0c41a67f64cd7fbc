import json, sys
for b in ["vec", "bs", "img", "ml", "hits", "dl"]:
    try:
        d = json.load(open(f"gpurun_out/bench_{b}.json"))
    except Exception as e:
        print(b, "ERR", e); continue
    bl = d.get("baselines", {})
    print(f"{b:5s} par {d['value']:8.3f} ser {bl.get('serial_resident_ms',0):8.3f} graph {bl.get('graph_resident_ms',0):8.3f} | "
          f"e2e {d['e2e']['value']:8.2f} ser {bl.get('serial_stream_ms',0):8.2f} graph {bl.get('graph_stream_ms',0):8.2f} | "
          f"roof {d['roofline']['kernel']} {d['roofline']['frac'] or 0:.2f} work_roof {d['roofline']['dag_work_roofline_ms']:.3f} sched {d['scheduler']['sched_us_per_launch']:.1f}us clk {d['clocks']['sm_mhz']}")
