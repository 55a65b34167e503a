# A/B of the chunked host path's chunk count on C4 (e2e through ei_cost_grad_host, pinned host
# buffers), 2 repeats each
OUT=gpurun_out/swch; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for r in 1 2; do
  for k in 8 16 32; do
    x=$(EI_HOST_CHUNKS=$k timeout 600 python bench.py --config C4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(d['ms_per_step'], e['ms_per_step'], e['ms_mean'], e['value'])")
    echo "chunks $k: $x" >> $OUT/res.txt
  done
done
