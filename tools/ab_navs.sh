# A/B of a compile-time navs.cu variant (-D<flag>): C5 step phases for BASE and the flag, twice each
# usage (on the GPU box): bash tools/ab_navs.sh FLAG
set -e
OBJS="build/capi.o build/primitives.o build/edges.o build/edge_extract.o build/navs.o build/volumes.o build/verify.o build/validate.o build/tables.o build/rings.o build/rowplan.o build/devgen.o build/devmem.o build/hostio.o build/host_api.o build/io.o"
for flag in BASE "$1" BASE "$1"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr -D$flag -c paper_2502_00778_b200/csrc/navs.cu -o build/navs.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2502_00778_b200/lib/libdualmesh.so $OBJS
  echo "== $flag"
  python tools/profile_step.py --config C5 --steps 12 | tail -1
done
