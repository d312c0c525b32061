#!/usr/bin/env python
"""Summarise an .ncu-rep (one kernel launch) into a small text file for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/NAME.txt [--regions N]

Reads the report with `ncu -i ... --page raw --csv` / `--page source --csv` (no GPU needed).
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__sass_inst_executed_op_local_ld.sum",
    "smsp__sass_inst_executed_op_local_st.sum", "smsp__warps_eligible.avg.per_cycle_active",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "sm__cycles_elapsed.max",
]


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    nreg = int(sys.argv[sys.argv.index("--regions") + 1]) if "--regions" in sys.argv else 24
    raw = page(rep, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    lines = [f"# ncu summary of {rep.split('/')[-1]} (ncu --set full --clock-control none; one launch)"]
    kn = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
    if kn is not None:
        lines.append(f"kernel: {vals[kn]}")
    for key in KEYS:
        for h, u, v in zip(hdr, units, vals):
            if h == key:
                lines.append(f"{h} [{u}] = {v}")
    src = page(rep, "source")
    if len(src) > 3:
        h = src[1]
        data = src[2:]
        isrc, isam, iex = h.index("Source"), h.index("# Samples"), h.index("Instructions Executed")
        tot = sum(int(r[isam]) for r in data) or 1
        lines.append(f"\n# stall samples by SASS region ({len(data)} instructions, {tot} samples)")
        B = max(1, len(data) // nreg)
        for b in range(0, len(data), B):
            blk = data[b:b + B]
            s = sum(int(r[isam]) for r in blk)
            ex = sum(int(r[iex]) for r in blk)
            ops = {}
            for r in blk:
                tok = r[isrc].split()
                op = (tok[1] if tok[0].startswith("@") else tok[0]).split(".")[0]
                ops[op] = ops.get(op, 0) + 1
            top = ", ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:5])
            lines.append(f"sass[{b:5d}:{b + len(blk):5d}] samples {100 * s / tot:5.1f}%  warp-instr executed {ex:>12d}  {top}")
        # opcode mix (dynamic)
        mix = {}
        for r in data:
            tok = r[isrc].split()
            op = (tok[1] if tok[0].startswith("@") else tok[0]).split(".")[0]
            mix[op] = mix.get(op, 0) + int(r[iex])
        total = sum(mix.values()) or 1
        lines.append("\n# dynamic opcode mix (warp instructions)")
        for k, v in sorted(mix.items(), key=lambda x: -x[1])[:18]:
            lines.append(f"{k:10s} {v:>14d} {100 * v / total:5.1f}%")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:45]))


if __name__ == "__main__":
    main()
