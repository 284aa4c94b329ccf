#!/bin/bash
# round-2 first GPU pass: full gpu suite (incl. new scale parity), cfg1 parity tool
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q -s -p no:cacheprovider > gpurun_out/r02a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a_pytest.log
timeout 1500 python tools/parity_cfg1.py 100000 200000 --ref > gpurun_out/r02a_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/r02a_parity.log
