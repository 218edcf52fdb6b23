set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
C=paper_2511_03655_b200/lib/libirk.so
timeout 900 python tools/ab.py --libs cur=$C,shfl=$V/libirk_g8shfl.so,g4=$C@4 --configs 1,2:10000:64,2:10000:512 --reps 2 --out gpurun_out/ab_o.json > gpurun_out/ab_o.log 2>&1
cat gpurun_out/ab_o.log
