"""Summarise an ncu --set full report (one block per kernel launch): the
metrics DESIGN.md and bench.py's roofline cite.  usage: ncu_summary.py X.ncu-rep > out.txt"""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read (tex)"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->L1 bytes"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active", "IMMA pipe %"),
    # sm_100 names: legacy mma.sync issue share, tensor pipe (tcgen05) and TMEM/UTC activity
    ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active", "mma.sync IMMA issue %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active %"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor memory (TMEM) %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
]

def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print("-----")
        print("  kernel:", r[ix["Kernel Name"]][:110])
        for k, name in KEYS:
            if k in ix:
                print(f"  {name:24s} {r[ix[k]]} {units[ix[k]]}   [{k}]")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.25:
                    stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        print("  stalls (warps per issue):", ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)))

if __name__ == "__main__":
    main(sys.argv[1])
