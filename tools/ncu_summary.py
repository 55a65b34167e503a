"""Summarise an ncu report (run here, no GPU): key throughput, shared-memory, stall metrics.
    python tools/ncu_summary.py gpurun_out/x.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__inst_executed.sum",
        "sm__inst_executed.sum.per_cycle_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "dram__bytes_read.sum",
        "dram__bytes_write.sum", "launch__registers_per_thread", "sm__cycles_elapsed.avg"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[h.index("Kernel Name")][:60])
        for k in KEYS:
            if k in h:
                print("   %-70s %s %s" % (k, r[h.index(k)], units[h.index(k)]))
        st = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v > 0.05:
                    st.append((v, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        try:   # the shared-memory data pipe moves one 128-B wavefront per SM-cycle
            g = lambda k: float(r[h.index(k)].replace(",", ""))
            sm_cyc = g("sm__cycles_elapsed.avg") * 148   # B200: 148 SMs
            wf = g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum")
            lts = g("lts__t_bytes.sum") * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[h.index("lts__t_bytes.sum")]]
            print("   %-70s %.3f" % ("derived: shared-load wavefronts per SM-cycle", wf / sm_cyc))
            print("   %-70s %.3f" % ("derived: + L2 bytes (TMA fills, outputs) / 128 B per SM-cycle", (wf + lts / 128) / sm_cyc))
        except (ValueError, KeyError, ZeroDivisionError):
            pass
        print("   stalls/issue:", ", ".join("%s %.2f" % (n, v) for v, n in sorted(st, reverse=True)[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
