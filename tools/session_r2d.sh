set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1200 python tools/ab.py --libs cur=paper_2511_03655_b200/lib/libirk.so,bps5=$V/libirk_bps5.so,bps5r200=$V/libirk_bps5r200.so,bps4r240=$V/libirk_bps4r240.so,bps4=$V/libirk_bps4.so --configs 2 --reps 3 --out gpurun_out/ab_d.json > gpurun_out/ab_d.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_d.log
