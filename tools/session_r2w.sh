set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1200 python tools/ab.py --libs base=$V/libirk_base.so,new=paper_2511_03655_b200/lib/libirk.so,r255=$V/libirk_r255.so,r224=$V/libirk_r224.so --configs 2 --reps 3 --out gpurun_out/ab_w.json > gpurun_out/ab_w.log 2>&1
cat gpurun_out/ab_w.log
