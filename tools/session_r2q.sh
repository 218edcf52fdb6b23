set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1200 python tools/ab.py --libs base=$V/libirk_base.so,spec0=$V/libirk_spec0.so,specall=$V/libirk_specall.so --configs 1,2:10000:512,2:10000:2048,2:10000:4096,2:10000:6144,2:10000:8192,2:10000:12288 --reps 2 --calls 2 --out gpurun_out/ab_q.json > gpurun_out/ab_q.log 2>&1
cat gpurun_out/ab_q.log
timeout 900 python -m pytest tests -m gpu -q -k "g8_stage or config1 or henon or kepler or divergence or max_iters or zero_steps or mapping or local" > gpurun_out/pytest_q.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_q.log
