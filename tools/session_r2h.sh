set -x
mkdir -p gpurun_out
python tools/run_once.py --config 2 > gpurun_out/plain_g1q.log 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ens_g1q -c 1 -o gpurun_out/g1qh python tools/run_once.py --config 2 > gpurun_out/ncu_g1qh.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/g1qh.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/g1qh_src.csv 2>/dev/null
ncu -i gpurun_out/g1qh.ncu-rep --page raw --csv > gpurun_out/g1qh_raw.csv 2>/dev/null
python tools/run_once.py --config 1 > gpurun_out/plain_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ens_gs -c 1 -o gpurun_out/c1 python tools/run_once.py --config 1 > gpurun_out/ncu_c1.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/c1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c1_src.csv 2>/dev/null
ncu -i gpurun_out/c1.ncu-rep --page raw --csv > gpurun_out/c1_raw.csv 2>/dev/null
rm -f gpurun_out/c1.ncu-rep
