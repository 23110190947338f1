import csv, subprocess, sys
def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return [dict(zip(r[0], row)) for row in r[2:]]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "lts__t_sectors_op_write.sum", "launch__grid_size", "launch__registers_per_thread"]
for rep in sys.argv[1:]:
    for d in raw(rep):
        print("==", rep, d.get("Kernel Name", "")[:60])
        for k in keys[1:]:
            print("  ", k, d.get(k))
        st = [(k, v) for k, v in d.items() if "smsp__average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")]
        st = sorted([(k, float(v)) for k, v in st if v not in ("", "n/a")], key=lambda x: -x[1])[:6]
        for k, v in st: print("   stall", k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), round(v, 3))
