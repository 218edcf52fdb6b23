timeout 30 python tools/run_once.py --config 3 --mapping 9 --batch 601 --nsteps 100 2>&1 | tail -1 || exit 1
timeout 300 python -m pytest tests/test_gpu_dmma.py -x -q 2>&1 | tail -3
timeout 60 python tools/nb_map_ab.py --nsteps 1000 --batches 16384 --ns 6 2>&1 | tail -1
