set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1200 python tools/ab.py --libs ts4=paper_2511_03655_b200/lib/libirk.so,ts1=$V/libirk_ts1.so,ts2=$V/libirk_ts2.so,ts8=$V/libirk_ts8.so --configs 2,2:2500:262144 --reps 3 --out gpurun_out/ab_i.json > gpurun_out/ab_i.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_i.log
timeout 900 python -m pytest tests -m gpu -q -k "config2 or work_queue or chunked or henon or divergence or million or energy or local" > gpurun_out/pytest_i.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_i.log
