"""Turns the raw-page CSVs of scripts/ncu_round2.sh (gpurun_out/) into the tracked summaries
under profiles/ (runs here, no GPU needed) and refreshes profiles/k1_traffic.json."""
import csv, json, os, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.max", "sm__cycles_active.avg",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def load(path):
    if not os.path.exists(path):
        return None, None, []
    rows = [r for r in csv.reader(open(path)) if r]
    if len(rows) < 3:
        return None, None, []
    return rows[0], rows[1], rows[2:]


def summarize(name):
    hdr, units, rows = load(os.path.join(ROOT, "gpurun_out", name + ".csv"))
    if not rows:
        print("no data:", name)
        return None
    out, traffic = [], []
    for r in rows:
        d = dict(zip(hdr, r))
        out.append(d["Kernel Name"][:110])
        for k in KEYS:
            if k in d:
                out.append(f"    {k:88s} {d[k]:>18s} {units[hdr.index(k)]}")
        if d["Kernel Name"].find("hybrid_") >= 0 or d["Kernel Name"].find("clenshaw_step") >= 0:
            tb = lambda k: float(d[k].replace(",", "")) * UNIT[units[hdr.index(k)]]
            traffic.append((d["Kernel Name"].split("(")[0], tb("dram__bytes_read.sum") + tb("dram__bytes_write.sum")))
    open(os.path.join(ROOT, "profiles", name + ".txt"), "w").write("\n".join(out) + "\n")
    return traffic


if __name__ == "__main__":
    traffic = {}
    for w in ("c3", "c4", "c2"):
        for tag in ("", "_warm"):
            t = summarize(f"r02_prof_k1_{w}{tag}")
            if t and not tag:
                # one Clenshaw step = one launch of every K1 kernel of the matrix: sum per kernel name
                per = {}
                for k, v in t:
                    per.setdefault(k, []).append(v)
                traffic[w] = sum(sum(v) / len(v) for v in per.values())
    for k in ("k3", "k4", "k6", "k8"):
        summarize(f"r02_prof_{k}_c3")
    path = os.path.join(ROOT, "profiles", "k1_traffic.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    old.update(traffic)
    json.dump(old, open(path, "w"), indent=1)
    print(old)
