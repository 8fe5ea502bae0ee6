"""Summarise ncu output for profiles/.
  python tools/ncu_summary.py rep  <file.ncu-rep> <title>     -> key metrics + stall samples
  python tools/ncu_summary.py launches <launches.csv> <title> -> per-kernel launch totals and shares
"""
import csv, io, subprocess, sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "smsp__sass_inst_executed_op_global_ld.sum",
        "smsp__sass_inst_executed_op_global_st.sum"]


def rep(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"# {title}")
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"{'Kernel Name':70s} {d.get('Kernel Name', '?')[:90]}")
        for k in KEYS:
            if k in d:
                print(f"{k:70s} {d[k]} {u.get(k, '')}")
        print("# warp-state samples")
        st = [(k, float(v)) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
              and v.replace('.', '', 1).isdigit()]
        for k, v in sorted(st, key=lambda t: -t[1]):
            if v > 0:
                print(f"{k:70s} {int(v)}")


def launches(path, title):
    text = open(path).read()
    i = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[i:])))
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
        tot[r["Kernel Name"]] += ms
        cnt[r["Kernel Name"]] += 1
    all_ms = sum(tot.values())
    print(f"# {title}")
    print("# launches  total_ms  share  kernel")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{cnt[k]:4d} {tot[k]:10.3f} {100 * tot[k] / all_ms:5.1f}%  {k[:110]}")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
