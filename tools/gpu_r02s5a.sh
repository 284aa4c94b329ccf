#!/bin/bash
# session 5, call a: k_win_cta resident-CTA A/B (lib/v5 = -DWC_MINB=5), e2e timing in and out of bench.py
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out; O=gpurun_out
for i in 1 2; do
  timeout 600 python tools/fp_time.py 795000000 4 2>&1 | tail -1 | sed 's/^/minb4: /' | tee -a $O/s5a_fp.log
  QS_LIB_PATH=$PWD/paper_1803_09835_b200/lib/v5/libquakescan_b200.so timeout 600 python tools/fp_time.py 795000000 4 2>&1 | tail -1 | sed 's/^/minb5: /' | tee -a $O/s5a_fp.log
done
QS_LIB_PATH=$PWD/paper_1803_09835_b200/lib/v5/libquakescan_b200.so timeout 600 python -m pytest tests/test_fingerprint_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2 | tee -a $O/s5a_fp.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-fingerprint --full-steps 0 --e2e-steps 3 > $O/s5a_bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/s5a_bench.log'):
    if l.startswith('{'):
        j=json.loads(l); print('bench e2e', j['e2e']['seconds_per_step'], 'pageable', j['e2e']['pageable']['seconds_per_step'], 'ms/step', j['ms_per_step'])
PY
QS_E2E_SPLITS=0.7 timeout 900 python tools/e2e_time.py 8000000 4 2>&1 | tail -4 | tee $O/s5a_e2e.log
