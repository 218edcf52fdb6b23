# round-2 session b: config-5 range pre-check (tests + timing), unit trace of the
# config-2 work queue, ncu source capture of the config-3 kernel
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "config5 or nbody_direct" > gpurun_out/pytest_c5.log 2>&1; echo c5 rc=$?
tail -3 gpurun_out/pytest_c5.log
timeout 300 python bench.py --steps 3 --warmup 3 --configs 5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_c5.json')); print(d['ms_per_step'], d['configs'])"
timeout 300 python tools/unit_trace.py > gpurun_out/unit_trace.log 2>&1; echo trace rc=$?
tail -40 gpurun_out/unit_trace.log
python tools/run_once.py --config 3 --nsteps 2000 > gpurun_out/plain_nb8.log 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ens_nbody8 -c 1 -o gpurun_out/nb8 python tools/run_once.py --config 3 --nsteps 2000 > gpurun_out/ncu_nb8.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/nb8.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/nb8_src.csv 2>/dev/null
ncu -i gpurun_out/nb8.ncu-rep --page raw --csv > gpurun_out/nb8_raw.csv 2>/dev/null
ls -la gpurun_out
