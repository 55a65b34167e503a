# A/B of a tuning knob on device-timed bench steps:  VAR=EI_K1_CLAIM VALS="1 0" CFGS="C2 P1" [REPS=3] [TESTS=1]
#   bash tools/dbg/ab.sh TAG
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ -n "${TESTS:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/res.txt
  tail -2 $OUT/pytest.log >> $OUT/res.txt
fi
for r in $(seq ${REPS:-3}); do for v in $VALS; do for c in $CFGS; do
  x=$(env $VAR=$v timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f' % (n[:2], v['ms']) for n, v in k.items()))")
  echo "$VAR=$v $c $x" >> $OUT/res.txt
done; done; done
