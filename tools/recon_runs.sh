#!/bin/bash
# NEXT-1 / NEXT-2 reconstructions on the GPU box (under gpurun): one JSON line each into
# gpurun_out/$TAG/recon.jsonl.  Usage: bash tools/recon_runs.sh TAG
set -u
TAG=${1:-recon}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_recon.log 2>&1 || exit 1
run() { timeout 900 python tools/reconstruct.py "$@" >> $OUT/recon.jsonl 2>> $OUT/recon.err; echo "recon $* rc=$?"; }
run --config C1 --noise 0 --iters 20000 --every 100
run --config C2 --noise 0 --iters 20000 --every 200
run --config C1 --noise 1 --stop discrepancy --iters 2000 --every 2
run --config C2 --noise 1 --stop discrepancy --iters 2000 --every 2
run --config C1 --noise 1 --iters 400 --every 20
run --config C4 --drift-slices 4 --noise 0 --iters 1000 --every 20
run --config C4 --drift-slices 4 --noise 1 --stop discrepancy --iters 1000 --every 5
run --config P1 --noise 0 --iters 5000
