#!/bin/bash
# Tests + smoke + all benches + ncu launch lists + overlap evidence.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
for b in ${BENCHES:-bs vec img ml hits dl}; do
  timeout 900 python bench.py --bench $b ${BENCH_ARGS} > gpurun_out/bench_$b.json 2> gpurun_out/bench_$b.err
done
for b in ${OVERLAP:-}; do
  timeout 600 python tools/overlap.py --bench $b --mode stream --out gpurun_out/overlap_${b}_stream.json > gpurun_out/overlap_$b.log 2>&1
  timeout 600 python tools/overlap.py --bench $b --mode resident --out gpurun_out/overlap_${b}_resident.json >> gpurun_out/overlap_$b.log 2>&1
done
for b in ${PROF:-}; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
     --clock-control none --csv --log-file gpurun_out/ncu_$b.csv python tools/profile_dag.py --bench $b --runs 2 > gpurun_out/ncu_$b.log 2>&1
done
tail -3 gpurun_out/pytest_gpu.log
