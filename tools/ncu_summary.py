#!/usr/bin/env python
"""Summarise an ncu report (--set full) into the numbers DESIGN.md / bench cite.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt

Prints per kernel: duration, instruction counts, IPC, issue-slot use,
occupancy, FP64 / DMMA / shared pipe utilisation, DRAM bytes (the
`traffic` of bench.py's roofline object), L1/L2 hit rates and the top warp
stall reasons (sampling).
"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration_ns"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc_per_sm"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "registers_per_thread"),
    ("launch__block_size", "block_size"),
    ("launch__grid_size", "grid_size"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_subpipe_pct"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared_pipe_fp64_plus_tensor_pct"),
    ("sm__inst_executed_pipe_fp64.sum", "fp64_pipe_instructions"),
    ("dram__bytes_read.sum", "dram_bytes_read"),
    ("dram__bytes_write.sum", "dram_bytes_write"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local_loads"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], dict(zip(rows[0], rows[1])), rows[2:]
    for r in data:
        d = dict(zip(hdr, r))
        print(f"kernel: {d.get('Kernel Name')}  grid {d.get('Grid Size')} block {d.get('Block Size')}")
        for k, name in KEYS:
            if k in d:
                print(f"  {name:36s} {d[k]} {units.get(k, '')}")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
              for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v}
        tot = sum(st.values()) or 1.0
        print("  top stall reasons (share of samples):")
        for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]:
            print(f"    {k:32s} {100 * v / tot:5.1f}%")
        print()


if __name__ == "__main__":
    main(sys.argv[1])
