# round-2 gpurun session: new GPU tests, full GPU suite, bench (all configs), ncu launch list
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_r2.py -m gpu -q -x > gpurun_out/pytest_r2.log 2>&1; echo r2 rc=$?
tail -3 gpurun_out/pytest_r2.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --configs none --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu rc=$?
