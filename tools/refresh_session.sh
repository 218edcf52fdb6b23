mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
python tools/run_once.py --config 2 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:ens_g1q -c 1 -o gpurun_out/g1q_full python tools/run_once.py --config 2 > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/g1q_full.ncu-rep --page raw --csv > gpurun_out/g1q_raw.csv 2>/dev/null
ncu -i gpurun_out/g1q_full.ncu-rep --page source --csv --print-source sass > gpurun_out/g1q_sass.csv 2>/dev/null
ls -la gpurun_out
