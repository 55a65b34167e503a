#!/bin/bash
# sweep tuning knobs on one config: bash tools/knobs.sh CFG "ENV1=a ENV2=b" "ENV1=c" ...
CFG=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for kv in "$@"; do
  env $kv python bench.py --config $CFG --no-cpu-baseline --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().splitlines()[-1]); k=d['kernels']
print('%-40s %.4f ms' % ('$kv', d['ms_per_step']), ' '.join('%s %.4f' % (n, v['ms']) for n, v in k.items()), d['plan'].get('k1_row_split'), d['plan'].get('k3_angle_split'))"
done
