# A/B of the FMA ring walk: C5 step phases BASE vs DM_RING_FMA (twice each), then the GPU parity
# tests on the FMA build.  usage (GPU box): bash tools/ab_fma.sh
bash tools/ab_navs.sh DM_RING_FMA
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr -DDM_RING_FMA -c paper_2502_00778_b200/csrc/navs.cu -o build/navs.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2502_00778_b200/lib/libdualmesh.so build/*.o
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
