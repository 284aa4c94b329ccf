#!/bin/bash
# session-5 evidence run on the final build (after the rolled drains): full gpu suite, default bench (both
# arms), launch list of bench.py itself, randomised sweeps, debug-assert build
# sweep, cfg3 run, full ncu captures of the top kernels
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out /tmp/ncu
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/s5e_pytest.log 2>&1; echo "pytest rc=$?" >> $O/s5e_pytest.log; tail -2 $O/s5e_pytest.log
timeout 1500 python bench.py > $O/s5e_bench.log 2> $O/s5e_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/s5e_bench_ref.log 2>&1; echo "ref rc=$?"
A='python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-fingerprint --full-steps 0'
timeout 900 $A > $O/s5e_bench_small.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"^k_|scan" --csv --log-file $O/s5e_bench_launches.csv $A > $O/s5e_ncu_list.log 2>&1; echo "list rc=$?"
python tools/launch_summary.py $O/s5e_bench_launches.csv --div 5 > $O/s5e_bench_launches.txt 2>&1; rm -f $O/s5e_bench_launches.csv; head -5 $O/s5e_bench_launches.txt
timeout 1200 python tools/stress_parity.py 150 > $O/s5e_stress_parity.log 2>&1; echo "stress rc=$?"; tail -2 $O/s5e_stress_parity.log
timeout 1200 python tools/stress_fingerprint.py 40 > $O/s5e_stress_fp.log 2>&1; echo "stress fp rc=$?"; tail -2 $O/s5e_stress_fp.log
timeout 1800 python tools/cfg3_run.py > $O/s5e_cfg3.log 2>&1; echo "cfg3 rc=$?"; tail -3 $O/s5e_cfg3.log | cut -c1-400
for KS in "k_pairs_pc:tools/one_search.py" "k_win_cta:tools/prof_fp.py"; do
  K=${KS%%:*}; S=${KS##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -c 1 -o /tmp/ncu/s5e_prof_$K -f python $S > $O/s5e_prof_$K.log 2>&1; echo "$K rc=$?"
  ncu -i /tmp/ncu/s5e_prof_$K.ncu-rep --page details --csv > $O/s5e_prof_${K}_details.csv 2>&1
  ncu -i /tmp/ncu/s5e_prof_$K.ncu-rep --page raw --csv > $O/s5e_prof_${K}_raw.csv 2>&1
done
if [ -f paper_1803_09835_b200/lib/debug/libquakescan_b200.so ]; then
  export QS_LIB_PATH=$GRAFT_REPO_ROOT/paper_1803_09835_b200/lib/debug/libquakescan_b200.so
  timeout 1200 python tools/stress_parity.py 100 > $O/s5e_dbg_stress_parity.log 2>&1; echo "dbg stress rc=$?" | tee -a $O/s5e_dbg_stress_parity.log
  timeout 1200 python tools/stress_fingerprint.py 20 > $O/s5e_dbg_stress_fp.log 2>&1; echo "dbg fp rc=$?" | tee -a $O/s5e_dbg_stress_fp.log
  timeout 1200 python -m pytest tests/test_lsh_gpu.py tests/test_buckets_gpu.py tests/test_capi_search_gpu.py -q -x -p no:cacheprovider -k "not full_scale" > $O/s5e_dbg_pytest.log 2>&1; echo "dbg pytest rc=$?" | tee -a $O/s5e_dbg_pytest.log
fi
# pair-stage DRAM traffic of one search (bench.py's roofline.traffic reads profiles/traffic.json)
timeout 900 python tools/one_search.py > $O/s5e_one.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum -k regex:"^k_|scan" --clock-control none --csv --log-file $O/s5e_search_launches.csv python tools/one_search.py > $O/s5e_ncu_one.log 2>&1
python tools/launch_summary.py $O/s5e_search_launches.csv --half --traffic $O/s5e_traffic.json > $O/s5e_search_launches.txt 2>&1; rm -f $O/s5e_search_launches.csv; head -4 $O/s5e_search_launches.txt
