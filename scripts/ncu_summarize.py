"""Label ncu's launch list with the engine's launch groups and summarise per group.

    python scripts/ncu_summarize.py gpurun_out/launches.csv gpurun_out/ncu_seq.json OUT.json [sweep_report.json]

The launch list comes from `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv python scripts/ncu_driver.py ...`; the
last chain's specialised-kernel launches (ooc_jit_kernel, ooc_sweep_kernel) are matched in order with the
sequence the driver recorded. Per-launch times under ncu are cold-cache and serialised:
compare shares, not absolutes.
"""
import csv
import json
import sys


def main(csv_path, seq_path, out_path, sweep_report=None):
    rows = {}
    with open(csv_path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if not r["ID"].isdigit():
            continue
        e = rows.setdefault(int(r["ID"]), {"kernel": r["Kernel Name"], "grid": r["Grid Size"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3,
                 "MB": 1e6, "GB": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
                 "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "second": 1, "s": 1}[unit]
        e[r["Metric Name"]] = v * scale
    seq = json.load(open(seq_path))
    last = seq["last_chain"]
    jit = [rows[i] for i in sorted(rows) if rows[i]["kernel"] in ("ooc_jit_kernel", "ooc_sweep_kernel")]
    jit = jit[-len(last):]
    iters = 14 if seq["app"].startswith("miniflow") else None
    groups = {}
    for (pos, nl, nbytes), r in zip(last, jit):
        if iters and pos == 140:
            key = "fieldsum"
        elif iters:
            key = f"L{pos % iters + 1}" + (f"-L{pos % iters + nl}" if nl > 1 else "")
        else:
            key = f"pos{pos}+{nl}"
        g = groups.setdefault(key, {"launches": 0, "s": 0.0, "dram": 0.0, "metric": 0.0,
                                    "grid": r["grid"], "kernel": r["kernel"]})
        g["launches"] += 1
        g["s"] += r["gpu__time_duration.sum"]
        g["dram"] += r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"]
        g["smem"] = g.get("smem", 0.0) + 128.0 * r.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0.0)
        g["metric"] += nbytes
    total = sum(g["s"] for g in groups.values())
    out = {"source": f"ncu launch list {csv_path}; last chain of scripts/ncu_driver.py "
                     f"({seq['app']} {seq['n']}, fuse={seq['fuse']}); cold-cache serialised replay",
           "kernels": []}
    if sweep_report:  # bench.py pairs these bytes with its timings only for the same kernel sources
        out["gen_hashes"] = sorted({e["gen_hash"] for e in json.load(open(sweep_report)) if "gen_hash" in e})
    for k, g in sorted(groups.items(), key=lambda kv: -kv[1]["s"]):
        us = 1e6 * g["s"] / g["launches"]
        db = g["dram"] / g["launches"]
        out["kernels"].append({"kernel": g["kernel"], "group": k, "grid": g["grid"],
                               "launches": g["launches"], "us_per_launch": round(us, 1),
                               "dram_bytes_per_launch": int(db),
                               "metric_bytes_per_launch": int(g["metric"] / g["launches"]),
                               "dram_TBps": round(db / us / 1e6, 3),
                               "smem_bytes_per_launch": int(g.get("smem", 0.0) / g["launches"]),
                               "smem_TBps": round(g.get("smem", 0.0) / g["launches"] / us / 1e6, 3),
                               "share": round(g["s"] / total, 3)})
    with open(out_path, "w") as f:
        json.dump(out, f, indent=1)
    for k in out["kernels"]:
        print(k)


if __name__ == "__main__":
    main(*sys.argv[1:5])
