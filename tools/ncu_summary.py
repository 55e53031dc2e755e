"""Per-kernel key metrics of an ncu report (raw page): python tools/ncu_summary.py <rep>"""
import csv, subprocess, sys
csv.field_size_limit(1 << 30)
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-metric-instances", "details"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr, units = r[0], r[1]
for row in r[2:]:
    d = dict(zip(hdr, row))
    print("==", d.get("Kernel Name", "")[:60], d.get("launch__grid_size"), "x", d.get("launch__block_size"))
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
              "sm__cycles_elapsed.avg.per_second", "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "lts__t_sector_hit_rate.pct",
              "launch__registers_per_thread", "sass__inst_executed_per_opcode"]:
        if k in d:
            print("  ", k, d[k][:400], units[hdr.index(k)])
    for k in hdr:
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                if float(d[k]) > 0: print("   stall", k.split("stalled_")[1], d[k])
            except ValueError:
                pass
