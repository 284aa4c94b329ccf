#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02s_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s_pytest.log
timeout 600 python tools/pair_table_bench.py 30 4e9 > gpurun_out/r02s_pairtable.log 2>&1
bash tools/gpu_debugchecks.sh
