#!/bin/bash
# ncu launch lists (per-kernel duration + DRAM bytes) for each benchmark DAG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for b in ${BENCHES:-bs vec img ml hits dl}; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
     --clock-control none --csv --log-file gpurun_out/ncu_$b.csv python tools/profile_dag.py --bench $b --runs 2 > gpurun_out/ncu_$b.log 2>&1
done
