# One ncu --set full capture per hot kernel (short runs), after a plain run of the same command.
set -e
run() {  # name regex cmd...
  local name=$1 rx=$2; shift 2
  "$@" > gpurun_out/plain_$name.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$rx -c 1 -o gpurun_out/ncu_$name "$@" > gpurun_out/ncu_$name.log 2>&1 || true
}
# g1q: profiles/r1/ens_g1q_kepler_full.ncu-rep (full config 2)
run g8    ens_g8     python tools/run_once.py --config 2 --batch 4096 --nsteps 2000
run nbody ens_nbody_q python tools/run_once.py --config 3 --nsteps 2000
run chain ens_chain_q python tools/run_once.py --config 4 --nsteps 5000
run force nbd_force  python tools/run_once.py --config 5 --nsteps 3
run fo    ens_fo_q   python tools/fo_once.py
# raw metrics as CSV (small), then keep only a few reports so gpurun_out stays < 64 MiB
for n in g1q g8 nbody chain force fo; do
  [ -f gpurun_out/ncu_$n.ncu-rep ] && ncu -i gpurun_out/ncu_$n.ncu-rep --page raw --csv > gpurun_out/ncu_${n}_raw.csv 2>/dev/null || true
done
rm -f gpurun_out/ncu_g1q.ncu-rep gpurun_out/ncu_g8.ncu-rep gpurun_out/ncu_fo.ncu-rep
