set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1200 python tools/ab.py --libs b4r240=$V/libirk_b4r240.so,b4r200=$V/libirk_b4r200.so,b3r255=$V/libirk_b3r255.so,u16=$V/libirk_b4r240u16.so,u64=$V/libirk_b4r240u64.so --configs 2 --reps 3 --out gpurun_out/ab_e.json > gpurun_out/ab_e.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_e.log
