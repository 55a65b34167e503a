mkdir -p gpurun_out/tr
EI_NVCC_DEFS=-DEI_TRACE python -c "from paper_2202_08627_b200 import build; build.build(force=True)" > gpurun_out/tr/build.log 2>&1
for c in C2 P1; do timeout 300 python tools/dbg/step_trace.py $c 10 > gpurun_out/tr/step_$c.txt 2>&1; done
timeout 300 python tools/dbg/k3_trace.py C2 5 > gpurun_out/tr/k3_C2.txt 2>&1
timeout 300 python tools/dbg/k1_trace.py C2 5 > gpurun_out/tr/k1_C2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_hmodel.py -x -q -m gpu > gpurun_out/tr/hmodel.log 2>&1
python -c "from paper_2202_08627_b200 import build; build.build(force=True)" > gpurun_out/tr/build2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hmodel.py -x -q -m gpu > gpurun_out/tr/hmodel.log 2>&1
tail -2 gpurun_out/tr/hmodel.log
cat gpurun_out/tr/step_*.txt gpurun_out/tr/k3_C2.txt | head -80
