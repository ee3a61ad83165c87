timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/par.log 2>&1
tail -1 gpurun_out/par.log
for conf in C5 C3 C4 C5; do timeout 300 python tools/profile_step.py --config $conf --steps 4 2>&1 | tail -1 | grep -o '"volume_order.*'; done
