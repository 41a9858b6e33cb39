#!/bin/bash
# One GPU session: gpu tests, smoke, a short bench.  Every step bounded by `timeout`.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; print('smoke', g.smoke())" > gpurun_out/smoke.log 2>&1
tail -3 gpurun_out/smoke.log
if [ -z "$NO_BENCH" ]; then
  timeout 400 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
