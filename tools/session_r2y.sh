set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1200 python tools/ab.py --libs base=$V/libirk_base.so,new=paper_2511_03655_b200/lib/libirk.so --configs 1,3:10000,2:10000:4096,2:10000:8192,3:10000:2048 --reps 2 --out gpurun_out/ab_y.json > gpurun_out/ab_y.log 2>&1
cat gpurun_out/ab_y.log
timeout 900 python -m pytest tests -m gpu -q -k "g8_stage or config1 or nbody or config3 or henon or kepler" > gpurun_out/pytest_y.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_y.log
