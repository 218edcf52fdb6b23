# final measurement session: GPU tests, bench line, launch list, ncu --set full of the bench kernel
# and of the config-3 kernel, strong-scaling projection (profiles/r2)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo pytest rc=$?
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke_final.log 2>&1; echo smoke rc=$?; cat gpurun_out/smoke_final.log | tail -2
tail -3 gpurun_out/pytest_final.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
cat gpurun_out/bench_final.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 --configs none --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
python tools/run_once.py --config 2 > gpurun_out/plain_final.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ens_g1q -c 1 -o gpurun_out/g1q_final python tools/run_once.py --config 2 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
ncu -i gpurun_out/g1q_final.ncu-rep --page raw --csv > gpurun_out/g1q_final_raw.csv 2>/dev/null
rm -f gpurun_out/g1q_final.ncu-rep
timeout 600 bash tools/ncu_src.sh 3 2000 ens_nbody8m nb8m_final; echo ncu3 rc=$?
timeout 600 bash tools/ncu_src.sh 1 0 ens_gsm c1_g8m_final; echo ncu4 rc=$?
timeout 1200 python tools/strong_scaling.py gpurun_out/strong_scaling_final.json > gpurun_out/strong_scaling_final.log 2>&1; echo ss rc=$?
