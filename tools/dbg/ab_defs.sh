# A/B/C of compile-time defines on device-timed bench steps:
#   VARIANTS="-DEI_A|;|-DEI_B" CFGS="C4 C2" [REPS=2] bash tools/dbg/ab_defs.sh TAG
# (variants separated by '|'; ';' = the default build)
TAG=${1:-abd}; OUT=gpurun_out/$TAG; mkdir -p $OUT
IFS='|' read -ra VS <<< "$VARIANTS"
for r in $(seq ${REPS:-2}); do for v in "${VS[@]}"; do
  d=${v//;/}
  EI_NVCC_DEFS="$d" python -c "from paper_2202_08627_b200 import build; build.build()" > $OUT/build.log 2>&1
  for c in $CFGS; do
    x=$(EI_NVCC_DEFS="$d" timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f' % (n[:2], v['ms']) for n, v in k.items()))")
    echo "[$d] $c $x" >> $OUT/res.txt
  done
done; done
cat $OUT/res.txt
