run() { python tools/profile_step.py --config C3 --steps 12 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['plan']['colored'], round(d['elem_ms'],4), round(d['total_ms'],4))"; }
run base
DUALMESH_PLAN_COLOR=1 run color8
DUALMESH_PLAN_COLOR=1 DUALMESH_COLOR_ROUNDS=16 run color16
DUALMESH_PLAN_COLOR=1 DUALMESH_COLOR_ROUNDS=4 run color4
ncu --set full --import-source on --clock-control none -k regex:k_navs_ring_pipe --launch-skip 2 -c 1 -o gpurun_out/c3_morton_u2 python tools/profile_step.py --config C3 --steps 4 > gpurun_out/c3_morton_ncu.log 2>&1
