# A/B: K3B (2x2 pixel blocks on the quad layout, EI_K3_QUAD=1) vs the triple-layout K3; parity first
# (The variant this script switched on was removed after the measurement recorded in DESIGN.md §5
# "Measured and rejected"; its knob no longer exists, so both arms now run the same code.)
OUT=gpurun_out/abq; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { c=$1; shift; x=$(env "$@" timeout 90 python bench.py --config $c --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f'%(n[:2],v['ms']) for n,v in k.items()))"); echo "$c $* $x" | tee -a $OUT/res.txt; }
EI_K3_QUAD=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cost_grad_parity or drift_gradient" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
for r in 1 2; do
  for c in C4 C5; do run $c EI_NONE=1; run $c EI_K3_QUAD=1; done
done
