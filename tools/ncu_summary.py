"""Summarise an ncu report: key metrics + top stall reasons + hottest source lines.
    python tools/ncu_summary.py report.ncu-rep [--source N]
"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'launch__block_size',
        'launch__grid_size', 'smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'lts__t_sectors.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__cycles_elapsed.avg.per_second', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed_op_shared_atom.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum',
        'sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed_pipe_xu.sum']


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    h, units, vals = raw(rep)
    for v in vals:
        print("kernel:", v[h.index("Kernel Name")] if "Kernel Name" in h else "?")
        for k in KEYS:
            if k in h:
                print(f"  {k} = {v[h.index(k)]} {units[h.index(k)]}")
        st = []
        for i, x in enumerate(h):
            if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("_not_issued"):
                try:
                    st.append((float(v[i]), x.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(a for a, _ in st) or 1
        print("  stalls:", ", ".join(f"{n} {a / tot:.0%}" for a, n in sorted(st, reverse=True)[:8]))
    if "--source" in sys.argv:
        nlines = int(sys.argv[sys.argv.index("--source") + 1])
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        rows = [r for r in rows if r and r[0] != "Kernel Name"]
        if not rows:
            return
        hh = rows[0]
        try:
            ci = hh.index("Warp Stall Sampling (All Samples)")
        except ValueError:
            print(hh)
            return
        si = hh.index("Source")
        body = [r for r in rows[1:] if len(r) > ci]
        body.sort(key=lambda r: -float(r[ci] or 0))
        ei = hh.index("Instructions Executed")
        tot_i = sum(float(r[ei] or 0) for r in body)
        print(f"  total warp instructions {tot_i:.3e}")
        for r in body[:nlines]:
            print(f"  {r[ci]:>8} {float(r[ei] or 0):>12.3e}  {r[si][:100]}")
        if "--dump" in sys.argv:
            body.sort(key=lambda r: int(r[0], 16))
            for r in body:
                print(f"  {r[0][-5:]} {r[ci]:>7} {float(r[ei] or 0):>11.3e}  {r[si][:90]}")


if __name__ == "__main__":
    main()
