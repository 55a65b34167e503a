# A/B of a compile-time define on device-timed bench steps:  DEFS="-DEI_X" CFGS="P1 C3" [REPS=3]
#   bash tools/dbg/ab_build.sh TAG
TAG=${1:-abb}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for r in $(seq ${REPS:-3}); do for d in "" "$DEFS"; do
  EI_NVCC_DEFS="$d" python -c "from paper_2202_08627_b200 import build; build.build(force=True)" > $OUT/build.log 2>&1
  for c in $CFGS; do
    x=$(timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f' % (n[:2], v['ms']) for n, v in k.items()))")
    echo "[$d] $c $x" >> $OUT/res.txt
  done
done; done
