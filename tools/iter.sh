#!/bin/bash
# quick GPU iteration: build, parity tests (optional filter), one ncu --set full capture of a kernel
# on a prof_case config, bench lines for a few configs.
#   bash tools/iter.sh TAG "KREGEX" "PROFCASE ARGS" "C4 C3 C2" [pytest -k expr]
TAG=$1; KRE=$2; PC=$3; CFGS=$4; KEXPR=${5:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
if [ -n "$KEXPR" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $OUT/pytest.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; fi
echo "pytest rc=$?"; tail -2 $OUT/pytest.log
if [ -n "$KRE" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 1 -c 1 -o $OUT/prof python tools/prof_case.py $PC > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
fi
for c in $CFGS; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > $OUT/bench_$c.json 2>$OUT/bench_$c.err
  python -c "
import json;d=json.loads(open('$OUT/bench_$c.json').read().splitlines()[-1]);print('$c', d['ms_per_step'], ' '.join('%s %.4f %.3f'%(k,v['ms'],v.get('frac') or 0) for k,v in d['kernels'].items()))"
done
