# ncu --set full + SASS source export of one kernel of one config (plain run first).
# usage: bash tools/ncu_src.sh <config> <nsteps> <kernel-regex> <tag> [extra run_once args]
set -e
mkdir -p gpurun_out
python tools/run_once.py --config $1 --nsteps $2 ${@:5} > gpurun_out/plain_$4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$3 -c 1 -o gpurun_out/$4 python tools/run_once.py --config $1 --nsteps $2 ${@:5} > gpurun_out/ncu_$4.log 2>&1
ncu -i gpurun_out/$4.ncu-rep --page raw --csv > gpurun_out/$4_raw.csv 2>/dev/null
ncu -i gpurun_out/$4.ncu-rep --page source --csv --print-source sass > gpurun_out/$4_sass.csv 2>/dev/null
ncu -i gpurun_out/$4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$4_src.csv 2>/dev/null
rm -f gpurun_out/$4.ncu-rep
echo done $4
