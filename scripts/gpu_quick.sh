#!/bin/bash
# Smoke + GPU tests (each bounded) + A/B of the tree against ab/libscfa_head.so.
mkdir -p gpurun_out
timeout 100 python -c "import __graft_entry__ as g; print('smoke', g.smoke())" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 500 python -m pytest tests -m gpu -q -x --timeout 60 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
if [ -z "$NO_AB" ]; then bash scripts/ab_libs.sh tree ${AB_LIBS:-ab/libscfa_head.so} > gpurun_out/ab.txt 2>&1; cat gpurun_out/ab.txt; fi
