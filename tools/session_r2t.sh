set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "fpu or config4 or chain" > gpurun_out/pytest_t.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_t.log
V=paper_2511_03655_b200/lib/variants
timeout 1500 python tools/ab.py --libs cw0=$V/libirk_cw0.so,cwall=$V/libirk_cwall.so --configs 4:20000:256,4:20000:512,4:20000:1024,4:20000:2048,4:20000:4096 --reps 1 --calls 2 --out gpurun_out/ab_t.json > gpurun_out/ab_t.log 2>&1
cat gpurun_out/ab_t.log
