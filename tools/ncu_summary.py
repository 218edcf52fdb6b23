"""Summarise ncu --set full raw CSV exports (one kernel each) into a markdown table:
duration, FP64 instructions -> achieved FP64 FLOP/s (DFMA = 2, DMUL/DADD = 1),
FP64 pipe utilisation, DRAM traffic and bandwidth, occupancy, registers."""
import csv
import sys

PEAK_TF = 37.22496   # 148 SM x 64 FMA/clk x 2 x 1.965 GHz
HBM_GBS = 6548.2     # MEASURED_PEAKS.json copy bandwidth


def load(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    units = rows[1]
    v = rows[2]
    return {k: (v[i], units[i]) for i, k in enumerate(h)}


def num(d, k, default=0.0):
    try:
        val, unit = d[k]
        x = float(val.replace(",", ""))
    except (KeyError, ValueError):
        return default
    scale = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0, "Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}
    return x * scale.get(unit, 1.0)


print("| kernel | time | FP64 pipe % of active cycles | SM active % | DRAM bytes | DRAM GB/s (% of 6,548) | warps/SM | lanes/instr | regs |")
print("|---|---|---|---|---|---|---|---|---|")
for path in sys.argv[1:]:
    d = load(path)
    name = d.get("Kernel Name", ("?", ""))[0].split("(")[0].replace("void ", "")[:40]
    t = num(d, "gpu__time_duration.sum")
    dram = num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")
    act = 100 * num(d, "sm__cycles_active.avg") / max(num(d, "sm__cycles_elapsed.avg"), 1)
    print(f"| {name} | {t*1e3:.2f} ms | {num(d, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
          f"{act:.1f} | {dram/1e6:.1f} MB | {dram/t/1e9 if t else 0:.1f} ({100*dram/t/1e9/HBM_GBS if t else 0:.2f} %) | "
          f"{num(d, 'sm__warps_active.avg.per_cycle_active'):.1f} | "
          f"{num(d, 'smsp__thread_inst_executed_per_inst_executed.ratio'):.1f} | {num(d, 'launch__registers_per_thread'):.0f} |")
