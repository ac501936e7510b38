"""profiles/ncu_traffic.json from a full ncu capture of the solve kernel (run here, on the report
gpurun brought back): DRAM bytes per launch (the bench line's roofline.traffic) and the FP32 work
the kernel actually executed, from the SASS thread-instruction counters.

python tools/ncu_traffic.py gpurun_out/<tag>_full.ncu-rep <agents> <kernel> > profiles/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, agents, kernel = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    val = {}
    for name, unit, x in zip(h, u, v):
        try:
            f = float(x.replace(",", ""))
        except ValueError:
            continue
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(unit, 1.0)
        val[name] = f * scale if unit in ("Kbyte", "Mbyte", "Gbyte", "byte") else f
    rd, wr = val["dram__bytes_read.sum"], val["dram__bytes_write.sum"]
    ffma = val["smsp__sass_thread_inst_executed_op_ffma_pred_on.sum.per_cycle_elapsed"]
    fadd = val["smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed"]
    fmul = val["smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed"]
    peak = 2 * val["sm__sass_thread_inst_executed_op_ffma_pred_on.sum.peak_sustained"]
    clk = val["sm__cycles_elapsed.avg.per_second"] * 1e9 if val["sm__cycles_elapsed.avg.per_second"] < 1e6 \
        else val["sm__cycles_elapsed.avg.per_second"]
    flop_cyc = 2 * ffma + fadd + fmul
    out = {
        "kernel": kernel, "agents": agents, "horizon": 10,
        "source": f"{rep} (ncu --set full, 1 launch of tools/ncu_driver.py {agents} 10: records, no z*)",
        "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
        "dram_bytes_per_agent": (rd + wr) / agents,
        "algorithmic_bytes_per_agent": {"in": 224, "out": 140, "z_star_if_requested": 1040},
        "note": "DRAM traffic of one launch; the records the kernel writes are still in the 126 MB L2 when it ends",
        "executed_fp32_flop_per_cycle": flop_cyc,
        "executed_fp32_tflops": flop_cyc * clk / 1e12,
        "fp32_peak_flop_per_cycle": peak,
        "executed_fp32_frac_of_peak": flop_cyc / peak,
        "executed_note": "ncu SASS thread-instruction counters (2 FFMA + FADD + FMUL per cycle elapsed) of the same "
                         "capture: FP32 work the squads actually execute, incl. the padded 28-column matrix rows",
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
