#!/bin/bash
# Re-entry check on a fresh box: full -m gpu suite, compute-sanitizer over every
# asynchronous kernel family, then the 1-GPU bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02u_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02u_pytest.log
for tool in memcheck racecheck synccheck; do
  QS_SAN_N=1500 timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_run.py > gpurun_out/r02u_san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02u_san_$tool.log
done
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02u_bench.log 2> gpurun_out/r02u_bench.err
echo "bench rc=$?" >> gpurun_out/r02u_bench.err
