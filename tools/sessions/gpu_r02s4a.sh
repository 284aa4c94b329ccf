#!/bin/bash
# session-4 start: full gpu suite + default bench (both arms) on the re-created container's build
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s4a_smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s4a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s4a_pytest.log
tail -3 gpurun_out/s4a_pytest.log
timeout 1200 python bench.py > gpurun_out/s4a_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s4a_bench.log | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/s4a_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/s4a_bench_ref.log | cut -c1-300
