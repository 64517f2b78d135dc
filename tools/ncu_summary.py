"""Summarise an ncu report into profiles/ (text + per-query DRAM traffic).

    python tools/ncu_summary.py gpurun_out/prof_v10.ncu-rep --queries 2000 --tag r1_count [--config 2]

--config N also records each kernel's DRAM bytes per query under "cfgN" in
profiles/ncu_traffic.json (bench.py's roofline.traffic for that config).
"""
import argparse
import csv
import io
import json
import os
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem)"),
    ("launch__cluster_dim_x", "cluster size"),
    ("launch__grid_size", "grid size"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "shared atomic wavefronts"),
    ("smsp__inst_executed_op_shared_atom.sum", "shared atomic instructions"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait / issue"),
]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--queries", type=int, required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", type=int, default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    root = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles")
    out = [f"# ncu --set full --clock-control none summary ({a.tag}, batch of {a.queries} queries)", ""]
    traffic_path = os.path.join(root, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0]
        out.append(f"## {name}")
        vals = {}
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"- {label:24s} {r[i]} {units[i]}")
                vals[m] = (r[i], units[i])
        rb = float(vals["dram__bytes_read.sum"][0]) * UNIT.get(vals["dram__bytes_read.sum"][1], 1)
        wb = float(vals["dram__bytes_write.sum"][0]) * UNIT.get(vals["dram__bytes_write.sum"][1], 1)
        out.append(f"- dram bytes per query    {(rb + wb) / a.queries:.1f} B")
        out.append("")
        key = {"k_count_cluster": "k_count", "k_count_enc": "k_count", "k_count_tma": "k_count",
               "k_count_pg": "k_count", "k_rerank_async": "k_rerank", "k_rerank_i8": "k_rerank"}.get(name, name)
        if a.config is not None:
            traffic.setdefault(f"cfg{a.config}", {})[key] = {
                "dram_bytes_per_query": (rb + wb) / a.queries, "source": os.path.basename(a.report), "tag": a.tag}
    with open(os.path.join(root, f"{a.tag}_ncu.md"), "w") as fh:
        fh.write("\n".join(out) + "\n")
    if a.config is not None:
        with open(traffic_path, "w") as fh:
            json.dump(traffic, fh, indent=1, sort_keys=True)
    print("\n".join(out))


if __name__ == "__main__":
    main()
