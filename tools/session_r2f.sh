set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1500 python tools/ab.py --libs u16=$V/libirk_b4r240u16.so,u8=$V/libirk_b4r240u8.so,u12=$V/libirk_b4r240u12.so,b6u16=$V/libirk_b6u16.so,b5u16=$V/libirk_b5r200u16.so,cur=paper_2511_03655_b200/lib/libirk.so --configs 2,2:2500:262144,2:10000:32768 --reps 2 --out gpurun_out/ab_f.json > gpurun_out/ab_f.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_f.log
