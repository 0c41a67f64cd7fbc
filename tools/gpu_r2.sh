#!/bin/bash
# Round-2 GPU iteration: selected tests, smoke, the default bench (suite), kineto overlap.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -n "${TESTS}" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest ${TESTS} -m gpu -q --maxfail=30 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -n "${BENCH}" ]; then
  timeout 1500 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
fi
for b in ${OVERLAP:-}; do
  timeout 600 python tools/overlap_kineto.py --bench $b --mode stream --out gpurun_out/ovk_${b}_stream.json --trace gpurun_out/trace_${b}_stream.json > gpurun_out/ovk_$b.log 2>&1
  timeout 600 python tools/overlap_kineto.py --bench $b --mode resident --out gpurun_out/ovk_${b}_resident.json > gpurun_out/ovk_${b}_r.log 2>&1
done
eval "${EXTRA:-true}"
tail -30 gpurun_out/pytest_gpu.log 2>/dev/null; tail -3 gpurun_out/smoke.log
head -c 3000 gpurun_out/bench.json 2>/dev/null; tail -5 gpurun_out/bench.err 2>/dev/null
for b in ${OVERLAP:-}; do tail -3 gpurun_out/ovk_$b.log; done
