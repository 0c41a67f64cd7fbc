#!/bin/bash
# Full GPU round: tests, smoke, every bench line (with cpu_baseline), the
# reference arm, the ncu launch list of the bench command itself, per-DAG
# ncu launch lists, schedule overlap, --set full captures of the dominant
# kernels and the B&S FP64 op count.  Summarise with tools/collect_profiles.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed"
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --maxfail=20 > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
for b in ${BENCHES:-bs vec img ml hits dl}; do
  timeout 900 python bench.py --bench $b $BENCH_ARGS > gpurun_out/bench_$b.json 2> gpurun_out/bench_$b.err
done
[ -z "$SKIP_REF" ] && timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
[ -z "$SKIP_REF" ] && timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
# launch list of the bench command (default workload), serialised by ncu
[ -z "$SKIP_REF" ] && timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/ncu_benchcmd.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-baselines > gpurun_out/ncu_benchcmd.log 2>&1
for b in ${PROF:-bs vec img ml hits dl}; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_$b.csv \
    python tools/profile_dag.py --bench $b --runs 2 > gpurun_out/ncu_$b.log 2>&1
done
for b in ${OVERLAP:-bs vec img ml hits dl}; do
  timeout 600 python tools/overlap.py --bench $b --mode stream --out gpurun_out/overlap_${b}_stream.json > gpurun_out/overlap_$b.log 2>&1
  timeout 600 python tools/overlap.py --bench $b --mode resident --out gpurun_out/overlap_${b}_resident.json >> gpurun_out/overlap_$b.log 2>&1
done
for kb in ${FULL:-bs:k_bs_l3b2 img:k_blur ml:k_norm hits:k_spmv$ dl:k_conv1_r2b3 dl:k_conv2_tmang}; do
  b=${kb%%:*}; k=${kb##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${k}" -c 1 -f \
    -o gpurun_out/prof_${k} python tools/profile_dag.py --bench $b --runs 1 > gpurun_out/prof_${k}.log 2>&1
done
[ -z "$SKIP_REF" ] && timeout 600 ncu --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
  --clock-control none -k regex:"k_bs_l3b2" -c 3 --csv --log-file gpurun_out/fp64_bs.csv \
  python tools/profile_dag.py --bench bs --runs 1 > gpurun_out/fp64_bs.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
