set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r2s5.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_r2s5.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_r2s5.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke_r2s5.log
timeout 600 python bench.py > gpurun_out/bench_r2s5.json 2> gpurun_out/bench_r2s5.err; echo bench rc=$?
cat gpurun_out/bench_r2s5.json
