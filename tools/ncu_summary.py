"""Summarise ncu --set full reports into the key-metric text kept under profiles/.

usage: python tools/ncu_summary.py report.ncu-rep [...] > profiles/ncu_full_<tag>.txt"""
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], [dict(zip(r[0], x)) for x in r[2:]]


for rep in sys.argv[1:]:
    head, units, recs = rows(rep)
    unit = dict(zip(head, units))
    for d in recs:
        print(f"  Kernel Name = {d.get('Kernel Name', '')[:120]}")
        print(f"  source report = {rep}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {unit.get(k, '')}".rstrip())
        st = [(k, d[k]) for k in d if k.startswith("smsp__average_warps_issue_stalled_") and
              k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")]
        for k, v in sorted(st, key=lambda x: -float(x[1]))[:6]:
            print(f"  {k} = {v}")
        print("---")
