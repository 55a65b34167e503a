# A/B: K1 CTAs of 32 angles (EI_K1_X2=1: 16 consumer warps, 1 CTA per SM, one staged window for
# (The variant this script switched on was removed after the measurement recorded in DESIGN.md §5
# "Measured and rejected"; its knob no longer exists, so both arms now run the same code.)
# both 16-angle halves) vs the default 16-angle CTAs at 2 per SM; parity first
OUT=gpurun_out/abx2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { c=$1; shift; x=$(env "$@" timeout 90 python bench.py --config $c --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f'%(n[:2],v['ms']) for n,v in k.items()))"); echo "$c $* $x" | tee -a $OUT/res.txt; }
EI_K1_X2=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "project_parity or cost_grad_parity or dot" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
for r in 1 2; do
  for c in C4 C3 C5; do run $c EI_NONE=1; run $c EI_K1_X2=1; done
done
