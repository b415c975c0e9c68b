"""Hottest SASS lines of one kernel in an ncu report (source page, SASS view),
by warp-stall samples:
    python tools/ncu_hot.py report.ncu-rep regex:cp_small [skip] [n]"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--kernel-name", kern,
                          "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    r = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = r[0]
    ci = {k: i for i, k in enumerate(h)}
    rows = [x for x in r[1:] if len(x) == len(h) and x[0].startswith("0x")]
    s_col, i_col = ci["Warp Stall Sampling (All Samples)"], ci["Instructions Executed"]
    tot_s = sum(float(x[s_col] or 0) for x in rows)
    tot_i = sum(float(x[i_col] or 0) for x in rows)
    print(f"samples {tot_s:.0f}  warp instructions {tot_i:.0f}")
    rows.sort(key=lambda x: -float(x[s_col] or 0))
    reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot_r = {k: sum(float(x[ci[k]] or 0) for x in rows) for k in reasons}
    print("stall reasons (samples):", ", ".join(f"{k[6:]} {v:.0f}" for k, v in
                                              sorted(tot_r.items(), key=lambda kv: -kv[1]) if v > 0))
    for x in rows[:n]:
        top = sorted(((float(x[ci[k]] or 0), k[6:]) for k in reasons), reverse=True)[:2]
        why = " ".join(f"{k}:{v:.0f}" for v, k in top if v > 0)
        print(f'{x[ci["Address"]][-5:]} {float(x[s_col] or 0):7.0f} {float(x[i_col] or 0):8.0f}  '
              f'{x[ci["Source"]].strip()[:70]:70s} {why}')


if __name__ == "__main__":
    main()
