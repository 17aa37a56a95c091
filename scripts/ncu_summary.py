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


def record(rep, n_particles, kernel, out_json):
    """The step-kernel record bench.py reads (profiles/force_kernel_ncu.json):
    per-launch DRAM bytes and the DRAM / L1TEX / FP64-pipe fractions of the
    first captured launch in `rep`."""
    import json
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units, row = r[0], r[1], r[2]
    d = dict(zip(h, row))
    u = dict(zip(h, units))

    def num(k, scale_units=None):
        v = float(d[k].replace(",", ""))
        if scale_units:
            v *= scale_units.get(u.get(k, ""), 1.0)
        return v
    b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    t = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    rec = {"kernel": kernel, "n_particles": int(n_particles),
           "ncu_kernel_name": d.get("Kernel Name", "")[:120],
           "dram_bytes_per_launch": num("dram__bytes_read.sum", b) + num("dram__bytes_write.sum", b),
           "dram_read_bytes": num("dram__bytes_read.sum", b),
           "dram_write_bytes": num("dram__bytes_write.sum", b),
           "duration_ms": num("gpu__time_duration.sum", t),
           "dram_frac_of_peak": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") / 100,
           "l1tex_frac_of_peak": num("l1tex__throughput.avg.pct_of_peak_sustained_active") / 100,
           "fp64_pipe_frac": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100,
           "issue_active_frac": num("smsp__issue_active.avg.pct_of_peak_sustained_active") / 100,
           "registers": int(num("launch__registers_per_thread")),
           "source": f"ncu --set full --clock-control none ({rep.split('/')[-1]})"}
    try:
        old = json.load(open(out_json))
        old = old if isinstance(old, list) else [old]
    except (OSError, ValueError):
        old = []
    old = [o for o in old if not (o.get("n_particles") == rec["n_particles"]
                                  and o.get("kernel") == kernel)]
    json.dump(old + [rec], open(out_json, "w"), indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    mode, arg = sys.argv[1], sys.argv[2]
    if mode == "record":
        record(arg, *sys.argv[3:6])
    else:
        {"raw": raw, "stalls": stalls, "launches": launches}[mode](arg)
