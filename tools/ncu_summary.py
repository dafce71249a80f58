"""Summarise ncu reports (gpurun_out/*.ncu-rep, launch CSVs) into profiles/ (run here, no GPU)."""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")]}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = {"value": vals[i], "unit": units[i]}
    return d


def sass_mix(rep, top=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    cnt = {}
    for r in data:
        op = r[ix["Source"]].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        try:
            n = float(r[ix["Instructions Executed"]])
        except ValueError:
            n = 0.0
        cnt[o.split(".")[0]] = cnt.get(o.split(".")[0], 0.0) + n
    tot = sum(cnt.values()) or 1.0
    return {k: round(100 * v / tot, 2) for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])[:top]}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    agg = {}
    for r in rows[hdr + 1:]:
        if len(r) != len(h) or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        unit = r[h.index("Metric Unit")]
        v = float(r[h.index("Metric Value")].replace(",", ""))
        v = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit] * v
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    return {k: {"launches": a[0], "total_us": round(a[1], 1), "share": round(a[1] / tot, 4)}
            for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])}


if __name__ == "__main__":
    tag = sys.argv[1]
    res = {"tag": tag, "k1": raw(f"gpurun_out/{tag}_k1.ncu-rep"),
           "k1_sass_mix_pct": sass_mix(f"gpurun_out/{tag}_k1.ncu-rep"),
           "k2": raw(f"gpurun_out/{tag}_k2.ncu-rep"),
           "k2_sass_mix_pct": sass_mix(f"gpurun_out/{tag}_k2.ncu-rep"),
           "launches": launches(f"gpurun_out/{tag}_launches.csv")}
    json.dump(res, open(f"profiles/{tag}_ncu_summary.json", "w"), indent=1)
    k1 = res["k1"]
    byts = (float(k1["dram__bytes_read.sum"]["value"]) * (1e9 if k1["dram__bytes_read.sum"]["unit"] == "Gbyte" else 1e6)
            + float(k1["dram__bytes_write.sum"]["value"]) * (1e9 if k1["dram__bytes_write.sum"]["unit"] == "Gbyte" else 1e6))
    json.dump({"kernel": k1["kernel"], "dram_bytes_per_launch": byts, "source": f"profiles/{tag}_ncu_summary.json"},
              open("profiles/ncu_k1_traffic.json", "w"), indent=1)
    print(json.dumps(res, indent=1))
