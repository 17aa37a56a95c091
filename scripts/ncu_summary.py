"""Summaries of ncu reports/launch lists (run here, no GPU needed)."""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "launch__grid_size", "launch__shared_mem_per_block_dynamic"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    for row in r[2:]:
        d = dict(zip(h, row))
        print(d.get("Kernel Name", "")[:40])
        for k in KEYS:
            if k in d:
                print(f"   {k:62s} {d[k]}")


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    for row in r[2:]:
        d = dict(zip(h, row))
        st = {k: float(v) for k, v in d.items()
              if k.startswith("smsp__average_warp_latency_issue_stalled") and k.endswith(".ratio")
              and v not in ("", "n/a")}
        st = {k: v for k, v in st.items()}
        top = sorted(st.items(), key=lambda x: -x[1])[:8]
        print("stalls", d.get("Kernel Name", "")[:30])
        for k, v in top:
            print(f"   {k.replace('smsp__average_warp_latency_issue_stalled_', ''):40s} {v:.2f}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    dram = collections.defaultdict(float)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d.get("Metric Name", "gpu__time_duration.sum")
            if name.startswith("dram__bytes"):
                unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
                    d["Metric Unit"], 1)
                dram[d["Kernel Name"].split("(")[0]] += float(
                    d["Metric Value"].replace(",", "")) * unit
                continue
            if name != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                     "msecond": 1e3}.get(u, 1.0)
            agg[d["Kernel Name"].split("(")[0]].append(v * scale)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':32s} {'n':>5s} {'total us':>10s} {'mean us':>9s} {'max us':>9s} share"
          f"{'  DRAM MB/launch' if dram else ''}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        extra = f"  {dram[k] / len(v) / 1e6:10.1f}" if dram else ""
        print(f"{k:32s} {len(v):5d} {sum(v):10.1f} {sum(v)/len(v):9.2f} {max(v):9.2f} "
              f"{sum(v)/tot:6.1%}{extra}")


if __name__ == "__main__":
    mode, arg = sys.argv[1], sys.argv[2]
    {"raw": raw, "stalls": stalls, "launches": launches}[mode](arg)
