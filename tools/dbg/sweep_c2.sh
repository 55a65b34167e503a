# One-call knob sweep on C2 (device-timed step, 2 repeats each): default, then one knob at a time
OUT=gpurun_out/swc2; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { x=$(env "$@" timeout 300 python bench.py --config C2 --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"); echo "$* $x" >> $OUT/res.txt; }
for r in 1 2; do
  run EI_NONE=1
  for v in 4 5 6 8; do run EI_K3_KS=$v; done
  for v in 1 3 4; do run EI_K1_RS=$v; done
  run EI_K1_NST=3
  for v in 4 16; do run EI_K1_RC=$v; done
  for v in 32 110; do run EI_K2_SMEM_KB=$v; done
  run EI_K1_RT=64
done
