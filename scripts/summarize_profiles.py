"""Summarise the ncu evidence of one GPU call into profiles/ (tracked).

    python scripts/summarize_profiles.py r01            # gpurun_out/prof_*.ncu-rep, launches.csv, bench.log
    python scripts/summarize_profiles.py r02 r02_       # gpurun_out/r02_prof_*.ncu-rep, r02_launches.csv, ...

Captures: prof_spmm (config 3 SpMM), prof_upd (config 3's dominant 6-in / 4-out update),
prof_bsr (config 4 BSR-12 product), prof_gram (s = 64 CTA-tiled DMMA Gram), prof_updmma
(config 2 tensor-core block update), prof_gramwarp (config 2 per-warp Gram of a block with
itself), prof_plane (config 3's plane-marching SpMM), prof_tail / prof_vt (config 3's fused eGl-QMR tail and V~ kernels, qmr_tail.cu), prof_flat (config 4's Gl-BiCGStab (X, R) flat plan, flat_upd.cu), prof_planerow (config 3's Gl-BiCGStab product with a row operand), prof_small (config 1's single-CTA eGl-BiCG iteration kernel; a launch covers the
iterations between two polls). Reads gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum launch list of
`python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu`), gpurun_out/prof_*.ncu-rep
(`ncu --set full`) and gpurun_out/bench.log, and writes
profiles/<tag>_launches.csv, profiles/<tag>_ncu_summary.json, profiles/<tag>_bench.json,
profiles/traffic.json (per-launch DRAM traffic of the dominant kernel for bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__t_sector_hit_rate.pct", "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_op_dmma.sum",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(tag, pre=""):
    os.makedirs(PROF, exist_ok=True)
    spath = os.path.join(PROF, f"{tag}_ncu_summary.json")
    summary = json.load(open(spath)) if os.path.exists(spath) else {}  # later captures of a round update the file
    for name in ("spmm", "upd", "bsr", "gram", "updmma", "gramwarp", "small", "band", "plane", "tail", "vt", "flat", "planerow"):
        rep = os.path.join(OUT, f"{pre}prof_{name}.ncu-rep")
        if not os.path.exists(rep):
            continue
        v, u = ncu_raw(rep)
        summary[name] = {"kernel": v.get("Kernel Name")}
        for m in METRICS:
            if m in v:
                summary[name][m] = f"{v[m]} {u.get(m, '')}".strip()
        rd = to_bytes(v["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        wr = to_bytes(v["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        summary[name]["dram_bytes_per_launch"] = rd + wr
    json.dump(summary, open(spath, "w"), indent=1)
    tj = {"source": f"profiles/{tag}_ncu_summary.json (ncu --set full, one launch, cold cache)"}
    if "plane" in summary:  # config 3's SpMM is the plane-marching kernel since round 2
        tj["cfg3_egl_qmr_spmm"] = summary["plane"]["dram_bytes_per_launch"]
    elif "spmm" in summary:
        tj["cfg3_egl_qmr_spmm"] = summary["spmm"]["dram_bytes_per_launch"]
    if "tail" in summary:  # the fused 7-input / 5-output tail (qmr_tail.cu): the dominant kernel of the eGl-QMR step
        tj["cfg3_egl_qmr_dominant"] = summary["tail"]["dram_bytes_per_launch"]
    elif "upd" in summary:  # before the fused tail: the 6-input / 4-output update
        tj["cfg3_egl_qmr_dominant"] = summary["upd"]["dram_bytes_per_launch"]
    if len(tj) > 1:
        json.dump(tj, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    lc = os.path.join(OUT, f"{pre}launches.csv")
    if os.path.exists(lc):
        lines = [ln for ln in open(lc) if ln.startswith('"')]
        rows = list(csv.DictReader(io.StringIO("".join(lines))))
        with open(os.path.join(PROF, f"{tag}_launches.csv"), "w") as f:
            f.write("id,kernel,grid,block,ns\n")
            for r in rows:
                k = r["Kernel Name"].split("(")[0].replace(",", ";")
                f.write(f'{r["ID"]},{k},{r["Grid Size"].replace(",", " ")},{r["Block Size"].replace(",", " ")},{r["Metric Value"]}\n')
        # share of one solver iteration (the last complete iteration in the list)
        names = [r["Kernel Name"].split("(")[0] for r in rows]
        ends = [i for i, nm in enumerate(names) if "end_iter" in nm]
        if len(ends) >= 2:
            it = rows[ends[-2] + 1: ends[-1] + 1]
            tot = sum(float(r["Metric Value"]) for r in it)
            share = {}
            for r in it:
                k = r["Kernel Name"].split("(")[0]
                share[k] = share.get(k, 0.0) + float(r["Metric Value"])
            json.dump({"iteration_ns": tot, "share": {k: v / tot for k, v in sorted(share.items(), key=lambda x: -x[1])},
                       "ns": share}, open(os.path.join(PROF, f"{tag}_iteration_shares.json"), "w"), indent=1)
    bl = os.path.join(OUT, f"{pre}bench.log")
    if os.path.exists(bl):
        for ln in open(bl):
            if ln.startswith("{"):
                json.dump(json.loads(ln), open(os.path.join(PROF, f"{tag}_bench.json"), "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", sys.argv[2] if len(sys.argv) > 2 else "")
