set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1500 python tools/ab.py --libs base=$V/libirk_base.so,new=paper_2511_03655_b200/lib/libirk.so --configs 2,1,3:10000,4:20000,5:100 --reps 2 --out gpurun_out/ab_k.json > gpurun_out/ab_k.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_k.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_k.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_k.log
