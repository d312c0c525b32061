#!/usr/bin/env python
"""BASELINE config 4: neighbor-count sweep m = 10/20/30/40/60 at n = 2^20, matern15_isotropic, with the ncu counters
SURVEY 8(d) asks for (FP64 pipe, local-memory loads/stores, achieved occupancy, L2 / DRAM throughput, registers).

    python tools/msweep.py [--out profiles/r2_msweep.json]        (on the GPU box; needs ncu)

Timing comes from CUDA events in a run WITHOUT the profiler; the counters from a separate `ncu --metrics ...` run of
one resident-table launch per m (never a timing source).
"""
import argparse, csv, io, json, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

METRICS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
           "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def time_m(m, n, family):
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "time_kernel.py"), "--m", str(m), "--n", str(n),
                          "--family", family, "--reps", "6"], capture_output=True, text=True)
    line = [ln for ln in out.stdout.splitlines() if "median" in ln]
    if not line:
        return {"error": (out.stderr or out.stdout)[-300:]}
    ln = line[-1]
    ms = float(ln.split("median")[1].split("ms")[0])
    kern = ln.split("kernel=")[1].split(": median")[0]
    return {"kernel_ms": ms, "kernel": kern}


def ncu_m(m, n, family):
    # launches: 16 chunked launches of the first evaluation (DeviceProblem's default for tables >= 32 MB), then
    # resident-table launches -> skip 17, capture 1
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:vecchia_", "-s", "17", "-c", "1",
           "--csv", sys.executable, str(ROOT / "tools" / "time_kernel.py"), "--m", str(m), "--n", str(n), "--family", family,
           "--reps", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    rows = [r for r in csv.reader(io.StringIO(out.stdout)) if len(r) > 10]
    if len(rows) < 2:
        return {"error": (out.stderr or out.stdout)[-300:]}
    head = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(head, r))
        try:
            res[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            res[d["Metric Name"]] = d["Metric Value"]
        res.setdefault("units", {})[d["Metric Name"]] = d["Metric Unit"]
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "r2_msweep.json"))
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--family", default="matern15_isotropic")
    ap.add_argument("--ms", default="10,20,30,40,50,60")
    a = ap.parse_args()
    import bench
    res = {"n": a.n, "family": a.family, "what": "config 4 neighbor-count sweep; kernel_ms from CUDA events (no profiler), "
           "counters from one launch under ncu --metrics (resident table)", "sweep": {}}
    for m in [int(x) for x in a.ms.split(",")]:
        t = time_m(m, a.n, a.family)
        c = ncu_m(m, a.n, a.family)
        F = bench.algorithmic_flops(a.family, 2, 1, 3, m)["F_min"]
        if "kernel_ms" in t:
            t["obs_per_s"] = a.n / (t["kernel_ms"] * 1e-3)
            t["algorithmic_tflops"] = F * a.n / (t["kernel_ms"] * 1e-3) * 1e-12
            t["flops_per_obs"] = F
        res["sweep"][str(m)] = {**t, "ncu": c}
        print(m, json.dumps(res["sweep"][str(m)])[:400], flush=True)
    Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
