#!/bin/bash
# K1 pipeline sweep (GPU box): build with EI_K1_NST=$1, run bench configs at shared-memory budgets
#   bash tools/sweep_k1.sh NST "KB..." "CFG..."
NST=$1; KBS=$2; CFGS=$3
EI_NVCC_DEFS=-DEI_K1_NST=$NST python -c "from paper_2202_08627_b200 import build; build.build(force=True)" > /dev/null 2>&1
for kb in $KBS; do for c in $CFGS; do
  EI_K1_SMEM_KB=$kb timeout 300 python bench.py --config $c --no-cpu-baseline --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().splitlines()[-1]); k=d.get('kernels',{})
print('NST=$NST KB=$kb $c', d['ms_per_step'], 'K1', k.get('K1_project',{}).get('ms'), 'RC', d.get('plan',{}).get('k1_rows_per_chunk'))"
done; done
