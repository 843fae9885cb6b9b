#!/usr/bin/env python
"""Summarise an ncu --set full report of the SSA kernel into a text file.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_k1_full_summary.txt [events]

Prints: headline metrics (duration, issue-slot / FP64 / ALU / FMA pipe
utilisation, SIMT efficiency, occupancy, DRAM traffic), the SASS instruction
mix per loop iteration (one candidate event per lane), the warp-stall
breakdown, and the most-stalled instructions.
"""
import collections
import csv
import io
import re
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_issued.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__grid_size",
    "launch__block_size",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
]
STALLS = ["stall_wait", "stall_math", "stall_not_selected", "stall_selected", "stall_short_sb",
          "stall_branch_resolving", "stall_dispatch", "stall_no_inst", "stall_long_sb", "stall_mio", "stall_lg"]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    events = float(sys.argv[3]) if len(sys.argv) > 3 else None
    lines = [f"ncu report: {rep}"]
    raw = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    lines.append(f"kernel: {kname}")
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            lines.append(f"  {m:66s} {vals[i]:>20s} {units[i]}")
    rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    h = rows[1]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    ith = h.index("Thread Instructions Executed")
    sidx = {c: h.index(c) for c in STALLS if c in h}
    ops = collections.Counter()
    counts = []
    stall_tot = collections.Counter()
    stall_ins = []
    tot_th = 0
    for r in rows[2:]:
        if len(r) <= ia:
            continue
        try:
            n = int(float(r[ia] or 0))
        except ValueError:
            continue
        s = r[isrc].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", s).split()[0].split(".")[0] if s else "?"
        ops[op] += n
        counts.append(n)
        tot_th += int(float(r[ith] or 0))
        st = 0.0
        for c, i in sidx.items():
            v = float(r[i] or 0)
            stall_tot[c] += v
            st += v
        stall_ins.append((st, s))
    # the event loop's body: the per-instruction count that carries the most executed instructions
    # (count x multiplicity), so once-per-warp prologue instructions cannot win by being many
    mult = collections.Counter(c for c in counts if c > 0)
    it = max(mult, key=lambda c: c * mult[c])
    tot = sum(ops.values())
    lines.append("")
    lines.append(f"warp-iterations of the event loop (the per-instruction count carrying the most instructions): {it}")
    lines.append(f"warp instructions per loop iteration: {tot / it:.1f}   (SIMT: {tot_th / max(tot, 1):.2f} threads/inst)")
    if events:
        lines.append(f"events in launch: {events:.4g}  -> warp instructions per event: {tot / events:.3f}")
    lines.append("instruction mix per iteration:")
    for op, n in ops.most_common(24):
        lines.append(f"  {op:12s} {n / it:8.2f}")
    T = sum(stall_tot.values()) or 1
    lines.append("")
    lines.append("warp stall samples (share of all samples):")
    for c, v in stall_tot.most_common():
        lines.append(f"  {c:26s} {v / T:6.3f}")
    lines.append("")
    lines.append("most stalled SASS instructions (share of samples):")
    for st, s in sorted(stall_ins, reverse=True)[:15]:
        lines.append(f"  {st / T:6.3f}  {s[:90]}")
    text = "\n".join(lines) + "\n"
    with open(dst, "w") as f:
        f.write(text)
    print(text)


if __name__ == "__main__":
    main()
