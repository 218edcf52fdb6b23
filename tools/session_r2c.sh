# round-2 session c: g1q parking + one-predicate weight range (A/B vs HEAD), parity tests, unit trace
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -k "config1 or config2 or work_queue or g8_stage or nbody or kepler or chunked or henon or max_iters or divergence or million" > gpurun_out/pytest_c.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_c.log
timeout 1200 python tools/ab.py --libs base=paper_2511_03655_b200/lib/variants/libirk_base.so,nopark=paper_2511_03655_b200/lib/variants/libirk_nopark.so,new=paper_2511_03655_b200/lib/libirk.so --configs 2,1,3:10000,5:100 --reps 2 --out gpurun_out/ab_c.json > gpurun_out/ab_c.log 2>&1; echo ab rc=$?
cat gpurun_out/ab_c.log
timeout 300 python tools/unit_trace.py --out gpurun_out/unit_trace_park.json > gpurun_out/unit_trace_park.log 2>&1; echo trace rc=$?
head -8 gpurun_out/unit_trace_park.log; tail -1 gpurun_out/unit_trace_park.log
