# A/B of K1's angles per CTA (EI_K1_NSL: 4 slots = 16 angles, 2 slots = 8) on the small configs,
# with the row split / ray tile knobs around it; device-timed step and K1 time, 2 repeats
OUT=gpurun_out/swnsl; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() { c=$1; shift; x=$(env "$@" EI_PLAN_VERBOSE=1 timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline 2>>$OUT/plan.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernels']['K1_project']['ms'], d['kernels']['K3_backproject']['ms'])"); echo "$c $* $x" >> $OUT/res.txt; }
for r in 1 2; do
  for c in C2 P1 C1; do
    run $c EI_K1_NSL=4
    run $c EI_K1_NSL=2
    for rs in 1 2 4; do for rt in 32 64; do run $c EI_K1_NSL=2 EI_K1_RS=$rs EI_K1_RT=$rt; done; done
  done
done
