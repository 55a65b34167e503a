# One-call knob sweep on C4 (device-timed step): default, then one knob at a time
OUT=gpurun_out/swc4; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { x=$(env "$@" timeout 300 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"); echo "$* $x" >> $OUT/res.txt; }
for r in 1; do
  run EI_NONE=1
  run EI_K1_NST=3
  for v in 8 32; do run EI_K1_RC=$v; done
  for v in 32 110; do run EI_K2_SMEM_KB=$v; done
  run EI_K1_RT=32
  run EI_NONE=2
done
