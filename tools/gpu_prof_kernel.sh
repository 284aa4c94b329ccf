# one ncu --set full capture of the first launch matching $1 in tools/prof_buckets.py (or $2 script)
cd $GRAFT_REPO_ROOT
K=${1:-k_bin_sort}; S=${2:-tools/prof_buckets.py}; SKIP=${3:-0}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip $SKIP -c 1 -o gpurun_out/prof_$K -f python $S > gpurun_out/prof_$K.log 2>&1; echo ncu $?
ncu -i gpurun_out/prof_$K.ncu-rep --page details --csv > gpurun_out/prof_${K}_details.csv 2>/dev/null
ncu -i gpurun_out/prof_$K.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${K}_sass.csv; ncu -i gpurun_out/prof_$K.ncu-rep --page source --csv --print-source cuda > gpurun_out/prof_${K}_cuda.csv 2>/dev/null 2>/dev/null
ls -la gpurun_out/prof_$K*
