#!/bin/bash
# compute-sanitizer over the smoke call (memcheck, racecheck, synccheck) and memcheck over the
# golden / reference-API parity / QK preparation GPU tests (needs a GPU).
mkdir -p gpurun_out
# without the caching allocator every tensor is its own allocation, so memcheck sees an access
# past a tensor's end (scripts/scratch/san_probe.py: one deliberate overrun, reported)
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/san_smoke_$tool.txt 2>&1
  echo "smoke $tool rc=$?: $(tail -1 gpurun_out/san_smoke_$tool.txt)"
done
timeout 2000 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_golden.py \
  tests/test_gpu_api_parity.py tests/test_gpu_qk_prepare.py tests/test_gpu_api.py tests/test_gpu_attention.py \
  tests/test_gpu_errors.py tests/test_gpu_schedule.py tests/test_gpu_sharding.py tests/test_lm.py tests/test_lsh.py \
  -m gpu -q -x -p no:cacheprovider > gpurun_out/san_tests.txt 2>&1
echo "tests memcheck rc=$?: $(grep -E 'passed|failed' gpurun_out/san_tests.txt | tail -1); $(tail -1 gpurun_out/san_tests.txt)"
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_golden.py \
  tests/test_gpu_api_parity.py tests/test_gpu_schedule.py -q -p no:cacheprovider > gpurun_out/san_sync.txt 2>&1
echo "tests synccheck rc=$?: $(grep -E 'passed|failed' gpurun_out/san_sync.txt | tail -1); $(tail -1 gpurun_out/san_sync.txt)"
timeout 1200 compute-sanitizer --tool initcheck --print-limit 20 python -m pytest tests/test_gpu_golden.py \
  tests/test_gpu_api_parity.py -q -p no:cacheprovider > gpurun_out/san_init.txt 2>&1
echo "tests initcheck rc=$?: $(grep -E 'passed|failed' gpurun_out/san_init.txt | tail -1); $(tail -1 gpurun_out/san_init.txt)"
