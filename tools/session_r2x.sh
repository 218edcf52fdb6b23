set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1200 python tools/ab.py --libs base=$V/libirk_base.so,new=paper_2511_03655_b200/lib/libirk.so --configs 2,2:10000:32768,2:2500:262144 --reps 3 --out gpurun_out/ab_x.json > gpurun_out/ab_x.log 2>&1
cat gpurun_out/ab_x.log
timeout 900 python -m pytest tests -m gpu -q -k "config2 or work_queue or chunked or henon or divergence or max_iters or million or local or kepler or energy" > gpurun_out/pytest_x.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_x.log
