"""Run tools/microbench (on-chip roofline denominators) under the bench's nvidia-smi clock sampler
and write the result with its clock record:
    python tools/measure_peaks.py [out.json]        (default gpurun_out/peaks.json)
The committed copy is profiles/r02/peaks.json; bench.py reads `smem_lds128_gbs` from it as the
K1/K3 roofline peak (scaled to the bench's own median SM clock when the two clocks differ)."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(out):
    import bench
    exe = os.path.join(ROOT, "tools", "microbench")
    src = exe + ".cu"
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-O3", "-o", exe, src])
    sampler = bench.ClockSampler(0)
    time.sleep(0.5)
    t0 = time.time()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    t1 = time.time()
    sampler.stop()
    d = json.loads(r.stdout.strip().splitlines()[-1])
    clocks = sampler.summary(t0, t1)
    d["clocks"] = clocks
    # the SM clock: measured under load by a clock64 spin kernel (cycles / event time); nvidia-smi's
    # samples also see the idle gaps between the short launches, and the block-span figures
    # undercount when a launch's blocks do not all start at once (both kept as cross-checks)
    d["sm_mhz"] = d.get("sm_mhz_spin") or clocks.get("sm_mhz") or 1965.0
    for k in ("smem_lds128", "smem_lds64", "l2_read"):
        d[k + "_bytes_per_clk_per_sm"] = round(d[k + "_gbs"] * 1e9 / (d["sm_mhz"] * 1e6) / d["sms"], 2)
    d["nominal_smem_gbs_at_clock"] = round(128.0 * d["sms"] * d["sm_mhz"] * 1e6 / 1e9, 1)
    d["how"] = ("tools/microbench.cu: best of 5 CUDA-event-timed launches each; LDS.128 / LDS.64 "
                "conflict-free (4 CTAs x 256 threads per SM), L2 read of a 48 MB resident buffer "
                "(__ldcg, 40 passes), HBM read of 4 GiB (8 passes); SM clock from a "
                "clock64 spin kernel; nvidia-smi clocks sampled during the run")
    d["when"] = time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "peaks.json"))
