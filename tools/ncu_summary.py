"""Summarise an ncu --set full report: duration, DRAM traffic, pipes, stalls.

usage: python tools/ncu_summary.py gpurun_out/prof.ncu-rep [label] > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
]


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary: {label}")
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        print(f"\n## {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                print(f"{k:70s} {d[k]:>22s} {u.get(k, '')}")
        stalls = []
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(d[k].replace(",", "")), k))
                except ValueError:
                    pass
        tot = sum(x for x, _ in stalls) or 1.0
        print("warp-state samples (share):")
        for x, k in sorted(stalls, reverse=True)[:10]:
            print(f"  {100 * x / tot:5.1f}%  {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}")


if __name__ == "__main__":
    main()
