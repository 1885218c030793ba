"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/summarize_ncu.py gpurun_out/prof_1m.ncu-rep gpurun_out/prof_32k.ncu-rep \
        --launches gpurun_out/launches.csv --out profiles/round1

Writes <out>_ncu.md (human summary), <out>_launches.csv (the launch list) and
profiles/ncu_score_pass.json (per-launch DRAM traffic of the headline score
kernel, read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import re
import shutil
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU ex2) pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tcgen05 unit %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "TMEM ld/st inst %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "SMEM wavefronts read by tcgen05"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU inst %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA inst %"),
]
STALL_PREFIX = "smsp__average_warps_issue_stalled_"
STALL_SUFFIX = "_per_issue_active.ratio"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        res.append(d)
    return res


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    per = {}
    kern = None
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "Kernel Name":
            kern = r[1]
            kern = norm(kern)
            per[kern] = []
        elif kern and r and r[0].startswith("0x") and len(r) > 3:
            per[kern].append((int(r[2] or 0), r[1].strip()))
    return per


def norm(name):
    """Kernel names differ between ncu pages ('void pairwise_tc_kernel<0>(PairArgs)'
    on the raw page, 'void fkde_b200::pairwise_tc_kernel<(int)0>(fkde_b200::PairArgs)'
    on the source page): strip namespaces and template-argument casts."""
    return re.sub(r"\w+::", "", name).replace("(int)", "").strip()


def fnum(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--launches", action="append", default=[])
    ap.add_argument("--out", default="profiles/round1")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    md = ["# ncu summary (" + os.path.basename(a.out) + ")", "",
          "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
          "(tools/profile_round.sh).  Per-launch numbers are cold-cache and serialised under "
          "replay; use shares, not absolutes, against bench.py's CUDA-event timings.", ""]
    score_json = None
    for rep in a.reps:
        md.append(f"## {os.path.basename(rep)}")
        md.append("")
        kerns = raw(rep)
        sp = stalls(rep)
        for k in kerns:
            name = k.get("Kernel Name", "?")
            md.append(f"### `{name}`")
            md.append("")
            md.append("| metric | value |")
            md.append("|---|---|")
            for key, label in METRICS:
                if key in k:
                    md.append(f"| {label} (`{key}`) | {k[key]} {k['_units'].get(key, '')} |")
            md.append("")
            st = sorted(((fnum(v) or 0.0, key[len(STALL_PREFIX):-len(STALL_SUFFIX)])
                         for key, v in k.items()
                         if key.startswith(STALL_PREFIX) and key.endswith(STALL_SUFFIX)), reverse=True)
            if st:
                md.append("Warp stall reasons (warps stalled per issued instruction):")
                md.append("")
                md.append(", ".join(f"{nm} {v:.2f}" for v, nm in st[:9] if v > 0.005))
                md.append("")
            samples = sp.get(norm(name), [])
            tot = sum(s for s, _ in samples) or 1
            top = sorted(samples, reverse=True)[:8]
            if top:
                md.append("Top warp-stall sample sites (share of all samples):")
                md.append("")
                for s, ins in top:
                    md.append(f"- {100.0 * s / tot:5.1f}%  `{ins}`")
                md.append("")
            wl = re.match(r"prof_w(\d)", os.path.basename(rep))
            if ("pairwise_tc_kernel<0>" in norm(name) and "1m" in os.path.basename(rep)) or \
                    (wl and "pairwise_tc_kernel" in norm(name)):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
                rd = fnum(k.get("dram__bytes_read.sum"))
                wr = fnum(k.get("dram__bytes_write.sum"))
                if rd is not None and wr is not None:
                    rd *= scale.get(k["_units"].get("dram__bytes_read.sum", "byte"), 1)
                    wr *= scale.get(k["_units"].get("dram__bytes_write.sum", "byte"), 1)
                    js = {"kernel": name, "report": os.path.basename(rep),
                          "dram_bytes_per_launch": rd + wr,
                          "duration": k.get("gpu__time_duration.sum"),
                          "duration_unit": k["_units"].get("gpu__time_duration.sum")}
                    if wl:   # bench.py --workload K reads profiles/ncu_workloadK.json
                        with open(os.path.join(os.path.dirname(a.out), f"ncu_workload{wl.group(1)}.json"),
                                  "w") as f:
                            json.dump(js, f, indent=1)
                    else:
                        score_json = js
    for li, lf in enumerate(x for x in a.launches if os.path.exists(x)):
        suffix = "" if len(a.launches) == 1 else "_" + os.path.splitext(os.path.basename(lf))[0]
        shutil.copy(lf, a.out + suffix + "_launches.csv")
        # launch-time shares per kernel name
        rows = list(csv.reader(open(lf)))
        hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        hdr = rows[hdr_i]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        agg = {}
        for r in rows[hdr_i + 1:]:
            if len(r) > vi:
                v = fnum(r[vi])
                if v is not None:
                    nm = r[ki].split("(")[0]
                    agg[nm] = agg.get(nm, 0.0) + v
        tot = sum(agg.values()) or 1
        md.append(f"## Launch list share ({os.path.basename(lf)}: bench.py --steps 2, gpu__time_duration)")
        md.append("")
        md.append("| kernel | total | share |")
        md.append("|---|---|---|")
        for nm, v in sorted(agg.items(), key=lambda x: -x[1]):
            md.append(f"| `{nm}` | {v:.0f} | {100 * v / tot:.2f}% |")
        md.append("")
    with open(a.out + "_ncu.md", "w") as f:
        f.write("\n".join(md) + "\n")
    if score_json:
        with open(os.path.join(os.path.dirname(a.out), "ncu_score_pass.json"), "w") as f:
            json.dump(score_json, f, indent=1)
    print("wrote", a.out + "_ncu.md", "score json:", score_json)


if __name__ == "__main__":
    main()
