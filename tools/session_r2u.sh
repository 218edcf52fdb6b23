set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1500 python tools/ab.py --libs cur=$V/libirk_base.so,b5=$V/libirk_b5.so,b3=$V/libirk_b3.so,u24=$V/libirk_u24.so,u12=$V/libirk_u12.so --configs 2 --reps 2 --out gpurun_out/ab_u.json > gpurun_out/ab_u.log 2>&1
cat gpurun_out/ab_u.log
