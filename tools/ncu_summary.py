#!/usr/bin/env python
"""Summarise an ncu report (details page) into the lines we track in profiles/."""
import csv
import subprocess
import sys

KEEP = ('GPU Speed Of Light Throughput', 'Compute Workload Analysis', 'Occupancy',
        'Scheduler Statistics', 'Warp State Statistics', 'Memory Workload Analysis',
        'Launch Statistics', 'Instruction Statistics')
WANT = ('Duration', 'Elapsed Cycles', 'SM Frequency', 'DRAM Throughput', 'Memory Throughput',
        'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Compute (SM) Throughput',
        'Executed Ipc Active', 'Issue Slots Busy', 'SM Busy', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Mem Pipes Busy', 'One or More Eligible', 'No Eligible', 'Active Warps Per Scheduler',
        'Eligible Warps Per Scheduler', 'Warp Cycles Per Issued Instruction',
        'Avg. Active Threads Per Warp', 'Avg. Not Predicated Off Threads Per Warp',
        'Executed Instructions', 'Registers Per Thread', 'Block Size', 'Grid Size',
        'Achieved Occupancy', 'Theoretical Occupancy', 'Dynamic Shared Memory Per Block',
        'Static Shared Memory Per Block')


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    for row in rows[1:]:
        d = dict(zip(hdr, row))
        if d.get('Section Name') in KEEP and d.get('Metric Name') in WANT:
            print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name'][:45]:45s} {d['Metric Value']:>16s} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    if len(r) > 2:
        h, units, vals = r[0], r[1], r[2:]
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum",
                     "smsp__thread_inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                     "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                     "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                     "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                     "smsp__average_warp_latency_issue_stalled_short_scoreboard",
                     "smsp__pcsamp_warps_issue_stalled_short_scoreboard"):
            if name in h:
                i = h.index(name)
                for v in vals:
                    print(f"{'raw':40s} {name[:60]:60s} {v[i]:>16s} {units[i]}")


def traffic(path, key, regex, stripes):
    """Sum dram__bytes_read + dram__bytes_write over the captured launches
    whose kernel name matches `regex` and record it in
    profiles/ncu_traffic.json under `key` (config:kernel) with the stripes
    the capture covered (bench.py scales it per stripe)."""
    import json
    import re
    from pathlib import Path
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, vals = r[0], r[2:]
    ik, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    unit_r, unit_w = r[1][ir], r[1][iw]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot, nk = 0.0, 0
    for v in vals:
        if re.search(regex, v[ik]):
            tot += float(v[ir].replace(",", "")) * scale[unit_r] + float(v[iw].replace(",", "")) * scale[unit_w]
            nk += 1
    out = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
    db = json.loads(out.read_text()) if out.exists() else {}
    db[key] = {"dram_bytes": tot, "launches": nk, "stripes": int(stripes), "source": Path(path).name}
    out.write_text(json.dumps(db, indent=1) + "\n")
    print(key, db[key])


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5])
    else:
        main(sys.argv[1])
