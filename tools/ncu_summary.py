"""Summarise an ncu report: duration, pipes, stall breakdown, top stalled SASS lines.

usage: python tools/ncu_summary.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    rows = ncu_csv(rep, "--page", "raw")
    d = dict(zip(rows[0], rows[2]))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]
    for k in keys:
        print(f"{k:60s} {d.get(k)}")
    st = {}
    for k, v in d.items():
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            if x > 0:
                st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
    tot = sum(st.values())
    print("stalls:", ", ".join(f"{k} {100 * x / tot:.1f}%" for k, x in sorted(st.items(), key=lambda t: -t[1])[:9]))
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    h = src[1]
    data = src[2:]
    ia, isrc = h.index("Address"), h.index("Source")
    iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot = sum(float(r[iss] or 0) for r in data)
    ops, cnt = Counter(), Counter()
    for r in data:
        t = r[isrc].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += float(r[iss] or 0)
        cnt[op.split(".")[0]] += float(r[iex] or 0)
    print("samples by opcode:", [(k, round(100 * v / tot, 1)) for k, v in ops.most_common(10)])
    print("executed by opcode:", [(k, int(v)) for k, v in cnt.most_common(14)])
    order = sorted(range(len(data)), key=lambda i: -float(data[i][iss] or 0))[:top]
    for i in order:
        prev = data[i - 1][isrc].strip()[:50] if i else ""
        print(f"{data[i][ia][-5:]} {float(data[i][iss]) / tot * 100:5.1f}% ex={data[i][iex]:>9} "
              f"{data[i][isrc].strip()[:60]:60s} | prev: {prev}")


if __name__ == "__main__":
    main()
