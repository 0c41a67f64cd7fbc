#!/bin/bash
# One GPU round: tests, smoke, bench per benchmark (logs under gpurun_out/)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
for b in ${BENCHES:-bs vec img ml hits dl}; do
  timeout 900 python bench.py --bench $b ${BENCH_ARGS} > gpurun_out/bench_$b.json 2> gpurun_out/bench_$b.err
done
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for b in ${BENCHES:-bs vec img ml hits dl}; do echo "== $b"; head -c 600 gpurun_out/bench_$b.json; echo; tail -3 gpurun_out/bench_$b.err; done
