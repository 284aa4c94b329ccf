#!/bin/bash
# session 5, call h: final build (12-bit host narrowing): full gpu suite, default bench (both arms), smoke, debug-assert sweeps
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
date +%s > $O/s5h_times.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/s5h_pytest.log 2>&1; echo "pytest rc=$?" >> $O/s5h_pytest.log; tail -2 $O/s5h_pytest.log
date +%s >> $O/s5h_times.log
timeout 1500 python bench.py > $O/s5h_bench.log 2> $O/s5h_bench.err; echo "bench rc=$?"
date +%s >> $O/s5h_times.log
timeout 900 python bench.py --impl reference > $O/s5h_bench_ref.log 2>&1; echo "ref rc=$?"
date +%s >> $O/s5h_times.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/s5h_smoke.log 2>&1; tail -1 $O/s5h_smoke.log
bash tools/gpu_debugchecks.sh; for f in dbg_sanitize_run dbg_stress_parity dbg_stress_fp dbg_pytest; do tail -n 2 $O/$f.log; done
