"""One-screen summary of an ncu --set full capture (raw page): time, DRAM bytes, throughput,
pipe utilisation, occupancy, registers and warp-stall breakdown.
usage: python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt"""
import csv, io, re, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keep = re.compile(r"^(Kernel Name|gpu__time_duration.sum|dram__bytes_(read|write)\.sum|dram__throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed|sm__throughput.avg.pct_of_peak_sustained_elapsed|"
                  r"sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_(active|elapsed)|sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active|"
                  r"sm__pipe_(alu|fma|shared)_cycles_active.avg.pct_of_peak_sustained_active|sm__warps_active.avg.pct_of_peak_sustained_active|"
                  r"launch__(grid_size|block_size|registers_per_thread|shared_mem_per_block_dynamic)|lts__t_sector_hit_rate.pct|"
                  r"smsp__inst_executed.sum|sm__cycles_elapsed.avg|smsp__cycles_active.avg|"
                  r"smsp__average_warps_issue_stalled_[a-z_]+_per_issue_active.ratio|smsp__issue_active.avg.pct_of_peak_sustained_active)$")
for r in rows[2:]:
    print("=" * 100)
    for h, u, v in zip(hdr, units, r):
        if keep.search(h):
            print(f"{h:75s} {v:>20s} {u}")
