"""One-page text summary of an `ncu --set full` capture (sections, stall reasons, SASS
opcode mix with the TMA / cp.async evidence) for profiles/.

    python scripts/ncu_full_summary.py REPORT.ncu-rep "title line" > profiles/NAME.txt
"""
import collections
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, title):
    print(f"# {title}")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    keep = ("GPU Speed Of Light Throughput", "Launch Statistics", "Occupancy", "Scheduler Statistics",
            "Warp State Statistics", "Compute Workload Analysis", "Memory Workload Analysis")
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Section Name") in keep and d.get("Metric Name"):
            print(d["Section Name"], "|", d["Metric Name"], "=", d["Metric Value"], d["Metric Unit"])
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    d = dict(zip(rows[0], rows[2]))
    for k in rows[0]:
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "launch__registers_per_thread",
                 "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                 "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") or (
                "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio") and float(d[k] or 0) > 0.05):
            print("raw |", k, "=", d[k])
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    ops, stall, tot = collections.Counter(), collections.Counter(), 0
    for r in rows[2:]:
        if len(r) < len(h):
            continue
        t = r[idx["Source"]].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ex = int(r[idx["Instructions Executed"]] or 0)
        ops[op] += ex
        stall[op] += int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        tot += ex
    print("# SASS of the captured launch: executed warp-instructions by opcode (share), stall samples")
    for k, v in ops.most_common(16):
        print(f"sass | {k:8s} {v:11d} {v / max(tot, 1) * 100:5.1f}%  stall-samples {stall[k]}")
    print(f"sass | UTMALDG (tensor TMA) executed: {ops['UTMALDG']}; UBLKCP (bulk TMA) executed: {ops['UBLKCP']}; "
          f"LDGSTS (cp.async) executed: {ops['LDGSTS']}; SYNCS (mbarrier) executed: {ops['SYNCS']}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
