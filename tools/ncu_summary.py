#!/usr/bin/env python3
"""Summarise an `ncu --set full` capture of one bench step's layer (k_sbmm + k_finalize per
linear, STEP_ORDER qkv, o, gate_up, down) into profiles/: a markdown table and the per-launch
DRAM traffic JSON that bench.py reports as roofline.traffic.

    python tools/ncu_summary.py gpurun_out/v14_full.ncu-rep v14
"""

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINDS = ["qkv", "o", "gate_up", "down"]
SHAPES = {"qkv": "12288x4096", "o": "4096x4096", "gate_up": "22016x4096", "down": "4096x11008"}
ALG = {"qkv": 757072128, "o": 252707072, "gate_up": 1356005632, "down": 678265088}  # SURVEY §8(d) formula
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    sb = [r for r in data if "k_sbmm" in r[idx["Kernel Name"]]]
    fin = [r for r in data if "k_finalize" in r[idx["Kernel Name"]]]
    assert len(sb) == 4 and len(fin) == 4, (len(sb), len(fin))

    def val(r, m):
        v = float(r[idx[m]].replace(",", ""))
        return v * SCALE.get(units[idx[m]], 1)

    lines = [f"# ncu --set full, fused SBMM kernel {tag} (k_sbmm + k_finalize), bench.py --layers 3, layer-2 launches",
             "", "Command: `ncu --set full --clock-control none --import-source on -k regex:\"k_sbmm|k_finalize\" "
             "-s 16 -c 8 -o gpurun_out/" + tag + "_full python bench.py --layers 3 --steps 1 --warmup 1 --no-graph "
             "--quick --no-e2e`", "", "## k_sbmm", "",
             "| metric | unit | " + " | ".join(f"{k} {SHAPES[k]}" for k in KINDS) + " |",
             "|---|---|" + "---|" * 4]
    for m in METRICS:
        if m not in idx:
            continue
        lines.append(f"| {m} | {units[idx[m]]} | " + " | ".join(sb[i][idx[m]] for i in range(4)) + " |")
    lines += ["", "## traffic vs algorithmic bytes", "",
              "| launch | algorithmic GB | k_sbmm DRAM GB | ratio | k_finalize DRAM MB | k_sbmm us | k_finalize us |",
              "|---|---|---|---|---|---|---|"]
    traffic = {}
    for i, k in enumerate(KINDS):
        s = val(sb[i], "dram__bytes_read.sum") + val(sb[i], "dram__bytes_write.sum")
        f = val(fin[i], "dram__bytes_read.sum") + val(fin[i], "dram__bytes_write.sum")
        traffic[k] = {"dram_bytes": s + f, "k_sbmm_dram_bytes": s, "k_finalize_dram_bytes": f,
                      "algorithmic_bytes": ALG[k]}
        lines.append(f"| {k} | {ALG[k] / 1e9:.4f} | {s / 1e9:.4f} | {s / ALG[k]:.3f} | {f / 1e6:.2f} | "
                     f"{sb[i][idx['gpu__time_duration.sum']]} | {fin[i][idx['gpu__time_duration.sum']]} |")
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    js = {"source": f"profiles/{tag}_ncu_full.md (ncu --set full, one capture per launch type, layer 2 of "
                    "bench.py --layers 3)", "kernel": f"k_sbmm {tag} (+ k_finalize)", "launches": traffic,
          "mean_dram_bytes_per_launch": sum(t["dram_bytes"] for t in traffic.values()) / 4,
          "mean_algorithmic_bytes_per_launch": sum(ALG.values()) / 4}
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_traffic.json"), "w") as fh:
        json.dump(js, fh, indent=1)
    print("\n".join(lines[-6:]))


if __name__ == "__main__":
    main()
