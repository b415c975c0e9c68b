"""Rewrite the result-table rows of DESIGN.md §8b, README.md and BASELINE.md §4
from a directory of bench lines (bench_c{1..5}.json) — so that the three
tables always quote one measurement set.

    python tools/results_table.py profiles/r02/s4/final
"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PARITY = {"c1": "1.5e-7", "c2": "2.9e-7", "c3": "3.8e-7", "c4": "7.6e-8", "c5": "2.4e-8"}   # pytest -m gpu -s log
WHAT = {"c2": "n=3, dim 1e5, 10M nnz, R=32 (headline)", "c3": "n=3, dim 1e6, 50M nnz Zipf, R=32",
        "c4": "n=4, dim 1e4, 20M nnz, R=16", "c5": "n=5, dim 1e3, 10M nnz, R=16"}


def fmt_bytes(b):
    return f"{b / 1e9:.2f} GB" if b >= 1e9 else f"{b / 1e6:.0f} MB"


def main():
    d = sys.argv[1]
    rows = {}
    for c in ("c1", "c2", "c3", "c4", "c5"):
        with open(os.path.join(ROOT, d, f"bench_{c}.json")) as f:
            rows[c] = json.load(f)

    def sub(path, pattern, repl):
        with open(os.path.join(ROOT, path)) as f:
            s = f.read()
        s2, n = re.subn(pattern, lambda m: repl, s, count=1, flags=re.M)
        assert n == 1, (path, pattern)
        with open(os.path.join(ROOT, path), "w") as f:
            f.write(s2)

    for c, b in rows.items():
        r = b["roofline"]
        ms, g, eff, of8 = b["ms_per_step"], b["value"] / 1e9, b["eff_gbs"], b["frac_of_8tbs"]
        kind = "reductions" if r["binding_op"].startswith("red.") else "mix"
        frac = f"{r['frac']:.2f} ({kind})"
        e2e = b["e2e"]["ms_per_step"]
        e2e_s = f"{e2e:.2f} ms" if e2e < 10 else f"{e2e:.1f} ms"
        cpu = b["cpu_baseline"]["value"] / 1e6
        cpu_s = f"{cpu:.1f} M nnz/s" if cpu >= 1 else f"{cpu:.2f} M nnz/s"
        if c == "c1":
            sub("DESIGN.md", r"^\| c1 \| \d[^\n]*$",
                f"| c1 | {ms:.3f} | {g:.2f} | {eff:.0f} | — | — (latency-bound: 2k nnz) | — | {e2e:.2f} ms | {PARITY[c]} |")
            sub("BASELINE.md", r"^\| c1 \| \d[^\n]*$",
                f"| c1 | {ms:.3f} | {g:.2f} | {eff:.0f} | — (latency-bound) | — | — | — | {PARITY[c]} | {e2e:.2f} ms | {cpu_s} |")
            continue
        traffic = fmt_bytes(r["traffic"])
        hb = r["hbm"]["frac_of_measured_copy_peak"]
        if c == "c2":
            sub("DESIGN.md", r"^\| \*\*c2\*\* \| [^\n]*$",
                f"| **c2** | **{ms:.3f}** | **{g:.2f}** | **{eff:.0f}** | **{of8:.2f}** | **{frac}** | {traffic} | {e2e_s} | {PARITY[c]} |")
            sub("BASELINE.md", r"^\| \*\*c2\*\* \| [^\n]*$",
                f"| **c2** | **{ms:.3f}** | **{g:.2f}** | **{eff:.0f}** | **{of8:.2f}** | **{hb:.2f}** | **{r['frac']:.2f} (gather+red mix)** | {traffic} | {PARITY[c]} | {e2e_s} | {cpu_s} |")
            sub("README.md", r"^\| c2 \| [^\n]*$",
                f"| c2 | {WHAT[c]} | {ms:.3f} ms | {g:.1f} G | {eff:.0f} ({100 * of8:.0f} % of 8 TB/s) | {r['frac']:.2f} |")
        else:
            sub("DESIGN.md", rf"^\| {c} \| \d[^\n]*$",
                f"| {c} | {ms:.3f} | {g:.2f} | {eff:.0f} | {of8:.2f} | {frac} | {traffic} | {e2e_s} | {PARITY[c]} |")
            sub("BASELINE.md", rf"^\| {c} \| \d[^\n]*$",
                f"| {c} | {ms:.3f} | {g:.2f} | {eff:.0f} | {of8:.2f} | {hb:.2f} | {frac} | {traffic} | {PARITY[c]} | {e2e_s} | {cpu_s} |")
            ms_s = f"{ms:.2f} ms" if ms >= 1 else f"{ms:.3f} ms"
            sub("README.md", rf"^\| {c} \| n=[^\n]*$", f"| {c} | {WHAT[c]} | {ms_s} | {g:.1f} G | {eff:.0f} | {r['frac']:.2f} |")
    pr = [rows[c]["timing"]["paper_rule"]["ms_min"] for c in ("c2", "c3", "c4", "c5")]
    print("paper rule (min) c2-c5: " + " / ".join(f"{x:.3f}" for x in pr))
    print("fractions: " + ", ".join(f"{c} {rows[c]['roofline']['frac']:.3f}" for c in ("c2", "c3", "c4", "c5")))
    print("clocks: " + ", ".join(f"{c} {rows[c]['clocks']['sm_mhz']:.0f} {rows[c]['clocks']['reasons']}" for c in rows))


if __name__ == "__main__":
    main()
