"""Summaries of an ncu --set full report: headline metrics, stall reasons,
per-source-line hot spots.  usage: ncu_summary.py report.ncu-rep [nlines]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nlines = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv", "--print-units", "base"))))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active"]
for w in want:
    if w in h:
        print(f"{w:70s} {v[h.index(w)]} {u[h.index(w)]}")
st = {n.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(v[i].replace(",", "") or 0))
      for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
tot = sum(st.values())
print("stall samples:", tot)
for k, c in sorted(st.items(), key=lambda kv: -kv[1])[:14]:
    print(f"   {k:28s} {c:7d} {100 * c / tot:5.1f}%")
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
per, text, cur = collections.Counter(), {}, None
for r in rows[3:]:
    if len(r) < 6:
        continue
    if r[0]:
        cur = r[0]
        text[cur] = r[1][:95]
    try:
        per[cur] += int(r[4] or 0)
    except ValueError:
        pass
t = sum(per.values()) or 1
print("hot source lines (% of stall samples):")
for ln, s in per.most_common(nlines):
    print(f"  {100 * s / t:5.1f}%  L{ln:>4}  {text.get(ln, '')}")
