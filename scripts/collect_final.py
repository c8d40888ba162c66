"""Copy the supporting lines of the round's final GPU call (scripts/gpu_r02_final2.sh) from
gpurun_out/ into profiles/ (tracked): the config 4 / config 1 bench lines, config 3 under the
other global methods, config 2's block-method table, and the A/B bench lines of the session.

    python scripts/summarize_profiles.py r02 r02_final_   # bench line, launch list, ncu summaries
    python scripts/collect_final.py                      # everything else
"""
import glob
import json
import os
import shutil

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(R, "gpurun_out")
PROF = os.path.join(R, "profiles")


def line(path):
    if not os.path.exists(path):
        return None
    for ln in open(path):
        if ln.startswith("{"):
            return json.loads(ln)
    return None


def kernels(d, n=7):
    return [{k: v for k, v in kk.items() if k in ("kernel", "avg_launch_ms", "frac", "share_of_step",
                                                    "algorithmic_bytes_per_launch")} for kk in d["iteration"]["kernels"]][:n]


def main():
    for cfg in ("cfg4", "cfg1"):
        d = line(os.path.join(OUT, f"r02_final_bench_{cfg}.log"))
        if d:
            json.dump(d, open(os.path.join(PROF, f"r02_bench_{cfg}.json"), "w"), indent=1)
    meth = {}
    for m in ("gl_bicgstab", "egl_bicg", "gl_qmr", "gl_bicg"):
        d = line(os.path.join(OUT, f"r02_final_bench_cfg3_{m}.log"))
        if d:
            meth[m] = {"value": d["value"], "unit": d["unit"], "ms_per_step": d["ms_per_step"],
                       "iteration_frac_of_hbm": d["iteration"]["frac_of_peak"], "kernels": kernels(d)}
    meth["note"] = ("config 3 (256^3, s = 16, FP64), the global methods besides the bench default eGl-QMR; "
                    "python bench.py --config 3 --method <m> --no-cpu --no-e2e (scripts/gpu_r02_final2.sh)")
    json.dump(meth, open(os.path.join(PROF, "r02_cfg3_methods.json"), "w"), indent=1)
    src = os.path.join(OUT, "r02_final_cfg2_methods.txt")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(PROF, "r02_cfg2_methods.txt"))
    ab = {}
    for f in sorted(glob.glob(os.path.join(OUT, "r02[fghijk]_bench*.log"))):
        d = line(f)
        if d:
            ab[os.path.basename(f)[:-4]] = {"value": d["value"], "ms_per_step": d["ms_per_step"],
                                            "kernels": [(k["kernel"], round(k["avg_launch_ms"], 3), k["frac"] and round(k["frac"], 3))
                                                        for k in d["iteration"]["kernels"]][:7]}
    ab["note"] = ("A/B bench lines of the round's last session (one gpurun call per prefix): r02f = eGl-QMR with / without "
                  "the vector fusion (SRK_NO_QMR_VEC_FUSE); r02g = flat plans / lean eGl-BiCG kernels vs the generic kernels "
                  "(SRK_NO_FLAT_UPDATE), config 3 and config 4; r02h = plane-marching SpMM row operands on / off "
                  "(SRK_NO_PLANE_ROWS), config 3 and config 2; r02i / r02j = Gl-BiCG flat plans; r02k = Gl-QMR flat plan")
    json.dump(ab, open(os.path.join(PROF, "r02_ab_lines.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
