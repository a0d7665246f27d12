# usage: bash tools/prof_one.sh <kernel-regex> <tag> [bench args...]
K=$1; TAG=$2; shift 2
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-6} -c 1 -o gpurun_out/$TAG python bench.py --no-cpu-baseline --steps 2 "$@" > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>/dev/null
ls -la gpurun_out/$TAG*
