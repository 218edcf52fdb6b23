set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_g.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_g.log
timeout 600 python bench.py > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; echo bench rc=$?
cat gpurun_out/bench_g.json
timeout 300 python tools/unit_trace.py --out gpurun_out/unit_trace_g.json > gpurun_out/unit_trace_g.log 2>&1; echo trace rc=$?
head -8 gpurun_out/unit_trace_g.log; tail -1 gpurun_out/unit_trace_g.log
