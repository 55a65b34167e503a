#!/bin/bash
# K1 staging sweep (GPU box): ring depth (EI_K1_NST, 2-4) x shared-memory budget (EI_K1_SMEM_KB)
# on bench configs; prints the step time, K1's time and the chunk size the plan chose.
#   bash tools/sweep_k1.sh "NST..." "KB..." "CFG..."
NSTS=$1; KBS=$2; CFGS=$3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in $NSTS; do for kb in $KBS; do for c in $CFGS; do
  EI_K1_NST=$n EI_K1_SMEM_KB=$kb timeout 300 python bench.py --config $c --no-cpu-baseline --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().splitlines()[-1]); k=d.get('kernels',{})
print('NST=$n KB=$kb $c', d['ms_per_step'], 'K1', k.get('K1_project',{}).get('ms'), 'RC', d.get('plan',{}).get('k1_rows_per_chunk'))"
done; done; done
