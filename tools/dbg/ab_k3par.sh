# A/B: K3 per-angle tables from the kernel-parameter bank (default) vs the staged records
# (The variant this script switched on was removed after the measurement recorded in DESIGN.md §5
# "Measured and rejected"; its knob no longer exists, so both arms now run the same code.)
# (EI_K3_SMEMTAB=1), device-timed step and per-kernel ms, 2 repeats
OUT=gpurun_out/abk3; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { c=$1; shift; x=$(env "$@" timeout 300 python bench.py --config $c --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f'%(n[:2],v['ms']) for n,v in k.items()))"); echo "$c $* $x" | tee -a $OUT/res.txt; }
for r in 1 2; do
  for c in C4 C3 C5 C2; do run $c EI_NONE=1; run $c EI_K3_SMEMTAB=1; done
done
