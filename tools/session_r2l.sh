set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
C=paper_2511_03655_b200/lib/libirk.so
timeout 1500 python tools/ab.py --libs auto=$C,g1=$C@1,g1b2=$V/libirk_bps2.so@1,g1b3=$V/libirk_bps3.so@1,g2=$C@2,g4=$C@4,g8=$C@8 --configs 2:10000:32768,2:10000:16384,2:10000:8192 --reps 1 --out gpurun_out/ab_l.json > gpurun_out/ab_l.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_l.log
