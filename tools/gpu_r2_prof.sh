#!/bin/bash
# Round-2 evidence job: full GPU tests, ncu launch lists of every DAG,
# ncu --set full of every product hot kernel, kineto overlap of every
# benchmark, compute-sanitizer on small parity tests.  Output: gpurun_out/$J/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
J=${J:-jx}
O=gpurun_out/$J
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
if [ -z "${SKIP_TESTS}" ]; then
  timeout 1800 python -m pytest tests -m gpu -q --maxfail=30 > $O/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
if [ -z "${SKIP_LAUNCH}" ]; then
  for b in ${BENCHES:-bs vec img ml hits dl}; do
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
       --clock-control none --csv --log-file $O/ncu_$b.csv python tools/profile_dag.py --bench $b --runs 2 > $O/ncu_$b.log 2>&1
  done
fi
# ncu --set full, one launch of each product hot kernel inside its DAG (the second run: warm)
for pair in ${FULL:-bs:k_bs2t_o6s3b2 hits:k_spmv_pad dl:k_conv2_h dl:k_conv1_r2b3 ml:k_nb_mmul ml:k_norm img:k_blur vec:k_square}; do
  b=${pair%%:*}; k=${pair##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:^${k}\$ -s 1 -c 1 \
     -o $O/prof_${k} python tools/profile_dag.py --bench $b --runs 2 > $O/prof_${k}.log 2>&1
done
for b in ${OVERLAP:-}; do
  timeout 600 python tools/overlap_kineto.py --bench $b --mode stream --out $O/ovk_${b}_stream.json > $O/ovk_$b.log 2>&1
  timeout 600 python tools/overlap_kineto.py --bench $b --mode resident --out $O/ovk_${b}_resident.json > $O/ovk_${b}_r.log 2>&1
done
if [ -n "${SANITIZE}" ]; then
  export PYTORCH_NO_CUDA_MEMORY_CACHING=1
  K="(img_parity or ml_parity or hits_parity or dl_parity or vec_parity or bs_parity) and not 1024 and not 200000 and not 100000 and not 515"
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python -m pytest tests/test_gpu_programs.py tests/test_gpu_vec_bs.py -m gpu -q -x -k "$K" > $O/sanitize_$tool.log 2>&1
    echo "rc=$?" >> $O/sanitize_$tool.log
  done
fi
eval "${EXTRA:-true}"
tail -5 $O/pytest_gpu.log 2>/dev/null; tail -2 $O/smoke.log
for f in $O/prof_*.log $O/sanitize_*.log; do echo "== $f"; tail -3 $f; done 2>/dev/null
