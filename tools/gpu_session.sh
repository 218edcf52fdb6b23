# one gpurun session: GPU tests, bench, full-size ncu capture of the bench kernel
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
python tools/run_once.py --config 2 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:ens_g1q -c 1 -o gpurun_out/g1q_full python tools/run_once.py --config 2 > gpurun_out/ncu.log 2>&1; echo ncu rc=$?
