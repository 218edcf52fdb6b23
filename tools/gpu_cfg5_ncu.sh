# ncu --set full of the config-5 force kernel (nbd_force, host-driven loop so every launch is visible)
# and the launch list of 20 config-5 steps (kernel shares of a sweep); round-2 close-out capture
set -x
mkdir -p gpurun_out
timeout 600 bash tools/ncu_src.sh 5 20 nbd_force cfg5_force_r2 --host-loop; echo ncu rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg5_r2.csv python tools/run_once.py --config 5 --nsteps 20 --host-loop > gpurun_out/ncu_cfg5_launch.log 2>&1; echo ncu2 rc=$?
