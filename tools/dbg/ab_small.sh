# Step times of the small configs (device-timed, ms), 3 repeats: C1 C2 P1 (and band on/off for P1)
OUT=gpurun_out/absmall; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { c=$1; shift; x=$(env "$@" timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f'%(n[:2],v['ms']) for n,v in k.items()), d.get('plan',{}).get('k1_band_rows'))"); echo "$c $* $x" | tee -a $OUT/res.txt; }
for r in 1 2 3; do
  for c in C1 C2 P1 C3; do run $c EI_NONE=1; done
  run P1 EI_K1_BAND=0
done
