# A/B of the working-tree navs.cu against HEAD's on the GPU box (same box, alternating):
# C5 step phases, twice each.  usage: bash tools/ab_head.sh [config]
set -e
CFG=${1:-C5}
git show HEAD:paper_2502_00778_b200/csrc/navs.cu > /tmp/navs_head.cu 2>/dev/null || cp tools/_navs_head.cu /tmp/navs_head.cu
cp /tmp/navs_head.cu paper_2502_00778_b200/csrc/navs_head.cu
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr"
$NV -c paper_2502_00778_b200/csrc/navs_head.cu -o /tmp/navs_head.o
$NV -c paper_2502_00778_b200/csrc/navs.cu -o /tmp/navs_new.o
rm paper_2502_00778_b200/csrc/navs_head.cu
OTHERS=$(ls build/*.o | grep -v '/navs.o')
for v in head new head new; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2502_00778_b200/lib/libdualmesh.so $OTHERS /tmp/navs_$v.o
  echo "== $v"
  python tools/profile_step.py --config $CFG --steps 12 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v,4) for k,v in d.items() if k.endswith('_ms')})"
  python tools/profile_step.py --config $CFG --steps 12 --algo traditional | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('trad', {k: round(v,4) for k,v in d.items() if k.endswith('_ms')})"
done
