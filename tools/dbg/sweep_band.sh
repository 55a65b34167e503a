# K1B band-mode sweep (device-timed step, ms): tile mode vs band mode at several band heights,
# on the small configs (C1, C2, P1).  Usage under gpurun: bash tools/dbg/sweep_band.sh [cfgs]
OUT=gpurun_out/swband; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { c=$1; shift; x=$(env "$@" timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f'%(n[:2],v['ms']) for n,v in k.items()), d.get('plan',{}).get('k1_band_rows'), d.get('plan',{}).get('k1_row_split'))"); echo "$c $* $x" | tee -a $OUT/res.txt; }
for c in ${*:-C2 C1 P1}; do
  for r in 1 2; do
    run $c EI_K1_BAND=0
    run $c EI_NONE=1
    for br in 6 8 11 12 16 20 24 32; do run $c EI_K1_BAND=1 EI_K1_BR=$br; done
  done
done
