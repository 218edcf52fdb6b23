set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
C=paper_2511_03655_b200/lib/libirk.so
timeout 1500 python tools/ab.py --libs g1=$C@1,g2=$C@2,g4=$C@4,g8=$C@8 --configs 2:10000:4096,2:10000:6144,2:10000:10240,2:10000:12288,2:10000:20480,2:10000:24576 --reps 1 --calls 2 --out gpurun_out/ab_m1.json > gpurun_out/ab_m1.log 2>&1
timeout 1500 python tools/ab.py --libs b4=$C@1,b2=$V/libirk_bps2.so@1,b3=$V/libirk_bps3.so@1 --configs 2:10000:24576,2:10000:40960,2:10000:49152,2:10000:57344 --reps 1 --calls 2 --out gpurun_out/ab_m2.json > gpurun_out/ab_m2.log 2>&1
cat gpurun_out/ab_m1.log gpurun_out/ab_m2.log
