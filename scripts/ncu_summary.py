"""Summarise ncu reports: key metrics per kernel + top stall reasons + hottest SASS lines.

    python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep [--sass N]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
]


def ncu(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 15
    rows = list(csv.reader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"=== [{d.get('ID')}] {d.get('Kernel Name', '')[:90]}")
        for k in KEYS:
            if k in d:
                print(f"    {k:70s} {d[k]:>16s} {units[hdr.index(k)]}")
    src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    out, h, kern = [], None, None
    for r in src:
        if r and r[0] == "Kernel Name":
            kern = r[1][:70]
            continue
        if r and r[0] == "Address":
            h = r
            continue
        if h and len(r) == len(h):
            d = dict(zip(h, r))
            d["kern"] = kern
            out.append(d)
    if not h:
        return
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    for kname in dict.fromkeys(d["kern"] for d in out):
        seen, uniq = set(), []
        for d in out:
            if d["kern"] != kname or d["Address"] in seen:
                continue
            seen.add(d["Address"])
            uniq.append(d)
        agg = {c: sum(int(d[c] or 0) for d in uniq) for c in cols}
        tot = sum(agg.values()) or 1
        print(f"--- stalls {kname}: " + ", ".join(f"{k[6:]} {100*v/tot:.0f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
        top = sorted(uniq, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:nsass]
        for d in top:
            print(f"    {int(d['Warp Stall Sampling (All Samples)']):6d}  {d['Source'][:100]}")


if __name__ == "__main__":
    main()
