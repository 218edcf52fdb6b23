set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "config1 or config2 or mapping or g8_stage or work_queue or kepler or henon" > gpurun_out/pytest_n.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_n.log
timeout 1200 python tools/strong_scaling.py gpurun_out/strong_scaling_r2.json > gpurun_out/strong_scaling.log 2>&1; echo ss rc=$?
cat gpurun_out/strong_scaling.log
