"""Summarise an ncu report (raw page) into the metrics DESIGN.md cites.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [...]     (or its `--page raw --csv` export)
    python tools/ncu_summary.py --json profiles/ncu_summary.json c2=raw.csv c3=raw.csv ...
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1_pct"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_read_sectors"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "l2_read_hit_sectors"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "red_requests"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "red_sectors"),
    ("lts__t_sectors_srcunit_tex_op_red.avg.pct_of_peak_sustained_elapsed", "red_sector_pct"),
    ("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "l2_atomic_input_pct"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "tma_bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_limit_smem"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall_lg_throttle"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall_not_selected"),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "stall_drain"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "stall_membar"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_short_sb"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "cycles_per_issue"),
]


def summarise(path):
    if path.endswith(".csv"):   # an exported raw page (ncu's log lines first)
        lines = open(path).read().splitlines()
        out = "\n".join(lines[next(i for i, l in enumerate(lines) if l.startswith('"ID"')):])
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for key, name in KEYS:
            if key in hdr:
                i = hdr.index(key)
                d[name] = (r[i], units[i])
        kn = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        res.append((kn, d))
    return res


def write_json(dst, pairs):
    """profiles/ncu_summary.json: DRAM bytes per launch of each config's MTTKRP kernel (bench.py `traffic`)."""
    import json
    res = {}
    for cfg, path in pairs:
        kn, d = next((k, d) for k, d in summarise(path) if "mttkrp_sym" in k)
        rd, wr = (float(d[k][0].replace(",", "")) for k in ("dram_read", "dram_write"))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale[d["dram_read"][1]]
        wr *= scale[d["dram_write"][1]]
        res[cfg] = {"dram_bytes_per_launch": int(round(rd + wr)),
                    "source": f"{path}: dram__bytes_read.sum {rd / 1e6:.6f} MB + dram__bytes_write.sum {wr / 1e6:.6f} MB "
                              f"({kn.split('(')[0].replace('void ', '').replace('systec::', '')}, ncu --set full --clock-control none)"}
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    if sys.argv[1:2] == ["--json"]:
        write_json(sys.argv[2], [a.split("=", 1) for a in sys.argv[3:]])
        sys.exit(0)
    for p in sys.argv[1:]:
        for kn, d in summarise(p):
            print(f"== {p}: {kn[:90]}")
            for k, (v, u) in d.items():
                print(f"   {k:22s} {v:>18s} {u}")
