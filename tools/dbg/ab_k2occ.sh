# K2 at 3 CTAs per SM (register cap 72, ring cap 64 KB) vs the default 2 (96 registers), C4 / C3
OUT=gpurun_out/abk2; mkdir -p $OUT
run() { d=$1; shift; c=$1; shift; x=$(env "$@" EI_NVCC_DEFS="$d" timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print(d['ms_per_step'], ' '.join('%s=%.4f/%.3f'%(n[:2],v['ms'],v.get('frac') or 0) for n,v in k.items()))"); echo "[$d] $c $* $x" | tee -a $OUT/res.txt; }
for r in 1 2; do
  for d in "" "-DEI_K2_MINB=3"; do
    EI_NVCC_DEFS="$d" python -c "from paper_2202_08627_b200 import build; build.build()" > $OUT/build.log 2>&1
    for c in C4 C3; do run "$d" $c EI_NONE=1; run "$d" $c EI_K2_SMEM_KB=64; run "$d" $c EI_K2_SMEM_KB=48; done
  done
done
python -c "from paper_2202_08627_b200 import build; build.build()"
