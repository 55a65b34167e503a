#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench lines for every config, ncu launch list of the
# default bench command and one `--set full` capture of K1/K3/K2.  Usage (under gpurun):
#   bash tools/gpu_round.sh TAG [what...]     what ⊂ {tests smoke bench ref ncu full peaks eicheck recon}
set -u
TAG=${1:-run}; shift || true
WHAT=${*:-tests smoke bench ncu full}
BENCH_CFGS=${BENCH_CFGS:-C4 C2 C1 C3 C5 P1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt 2>&1
nproc >> $OUT/gpu.txt; grep -m1 "model name" /proc/cpuinfo >> $OUT/gpu.txt
for w in $WHAT; do
  case $w in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?" | tee -a $OUT/rc.txt
      tail -3 $OUT/pytest_gpu.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/rc.txt
      tail -1 $OUT/smoke.log ;;
    bench)
      for c in $BENCH_CFGS; do
        timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?" | tee -a $OUT/rc.txt
        python - $OUT/bench_$c.json <<'EOF'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k = d.get("kernels", {})   # P1's line has no per-kernel split
    print(d["config"]["workload"][:3], "ms/step %.4f" % d["ms_per_step"], "e2e %.1f" % (d.get("e2e") or {}).get("value", 0.0),
          " ".join("%s %.4fms %.3f" % (n, v["ms"], v.get("frac", 0)) for n, v in k.items()))
except Exception as e:
    print("parse fail", e)
EOF
      done ;;
    ref)
      timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?" | tee -a $OUT/rc.txt
      tail -c 600 $OUT/bench_ref.json ;;
    eicheck)
      # the parity suite under a bounds-checking build (-DEI_CHECK: K3 checks every tap against its
      # staged window, K1 every chunk's extreme taps; ei_plan_info out[4] must stay 0), then the
      # normal build again
      EI_NVCC_DEFS=-DEI_CHECK python -c "from paper_2202_08627_b200 import build; build.build()" > $OUT/build_check.log 2>&1
      EI_NVCC_DEFS=-DEI_CHECK timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_limits.py -m gpu -x -q > $OUT/pytest_gpu_eicheck.log 2>&1
      echo "eicheck rc=$?" | tee -a $OUT/rc.txt; tail -2 $OUT/pytest_gpu_eicheck.log
      python -c "from paper_2202_08627_b200 import build; build.build()" >> $OUT/build.log 2>&1 ;;
    recon)
      # NEXT-1 / NEXT-2 full reconstructions (tools/recon_runs.sh) into $OUT/recon.jsonl
      bash tools/recon_runs.sh $TAG > $OUT/recon.log 2>&1; echo "recon rc=$?" | tee -a $OUT/rc.txt ;;
    peaks)
      timeout 600 python tools/measure_peaks.py $OUT/peaks.json > $OUT/peaks.log 2>&1; echo "peaks rc=$?" | tee -a $OUT/rc.txt
      tail -c 400 $OUT/peaks.json ;;
    ncu)
      # the launch list of the default bench command's timed steps (NVTX range "timed" in bench.py)
      timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/plain_launch.log 2>&1 &&
      timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
      echo "ncu launches rc=$?" | tee -a $OUT/rc.txt ;;
    full)
      # one --set full capture per config of the three hot kernels of one bench step (the 4th),
      # the source of profiles/traffic.json (tools/ncu_traffic.py) and the ncu summaries
      for c in ${FULL_CFGS:-C2 C3 C5 C4}; do
        timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $OUT/plain_full_$c.log 2>&1 &&
        timeout 900 ncu --set full --metrics lts__t_bytes.sum,l1tex__t_bytes.sum --clock-control none \
          --import-source on --kernel-name-base demangled --nvtx --nvtx-include "timed/" \
          -k regex:"project_kernel<\\(int\\)3|curve_kernel<\\(int\\)1>|backproject3_kernel" -c 3 \
          -o $OUT/full_$c python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$c.log 2>&1
        echo "ncu full $c rc=$?" | tee -a $OUT/rc.txt
      done ;;
  esac
done
