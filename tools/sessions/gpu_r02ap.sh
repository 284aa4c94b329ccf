#!/bin/bash
# Mid-session evidence: full -m gpu suite, 1-GPU bench (both arms), launch list of one cfg1 search
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02ap_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02ap_pytest.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02ap_bench.log 2> gpurun_out/r02ap_bench.err
echo "bench rc=$?" >> gpurun_out/r02ap_bench.err
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02ap_ref.log 2> gpurun_out/r02ap_ref.err
echo "ref rc=$?" >> gpurun_out/r02ap_ref.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum -k regex:"^k_|scan" --clock-control none --csv --log-file gpurun_out/r02ap_search_launches.csv python tools/one_search.py > gpurun_out/r02ap_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r02ap_ncu.log
