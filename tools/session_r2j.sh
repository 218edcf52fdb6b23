set -x
mkdir -p gpurun_out
V=paper_2511_03655_b200/lib/variants
timeout 1500 python tools/ab.py --libs base=$V/libirk_base.so,cur=paper_2511_03655_b200/lib/libirk.so,s512b128m7=$V/libirk_s512b128m7.so,s512b128m8=$V/libirk_s512b128m8.so,s512b256m3=$V/libirk_s512b256m3.so,m2=$V/libirk_s1024b256m2.so --configs 5:100 --reps 2 --out gpurun_out/ab_j.json > gpurun_out/ab_j.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_j.log
timeout 900 python -m pytest tests -m gpu -q -k "config5 or nbody_direct" > gpurun_out/pytest_j.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_j.log
