"""Key metrics per kernel of an `ncu --set full` report (text table for
profiles/): duration, DRAM bytes and GB/s, SM/L1/L2 throughput, IPC,
occupancy, registers, shared memory, top warp-stall reasons."""
import csv, io, subprocess, sys
rep = sys.argv[1]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
     "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_active",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
     "launch__shared_mem_per_block_static", "smsp__inst_executed.sum"]
ST = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "mio_throttle", "lg_throttle", "math_pipe_throttle",
      "selected", "not_selected", "no_instructions", "branch_resolving", "drain", "membar", "dispatch_stall"]
metrics = M + [f"smsp__pcsamp_warps_issue_stalled_{s}" for s in ST] + ["smsp__pcsamp_sample_count"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    f = lambda k: float(d[k].replace(",", "")) if d.get(k) not in (None, "", "n/a") else float("nan")
    t_us = f("gpu__time_duration.sum") / 1000.0 if f("gpu__time_duration.sum") > 1000 else f("gpu__time_duration.sum")
    name = d["Kernel Name"].split("(")[0]
    print(f"== {name}")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    print(f"   time {d['gpu__time_duration.sum']} (ncu unit)  grid {d['launch__grid_size']} x block {d['launch__block_size']}  "
          f"regs {d['launch__registers_per_thread']}  smem dyn {d['launch__shared_mem_per_block_dynamic']} static {d['launch__shared_mem_per_block_static']}")
    print(f"   dram read {rd:.4g}  write {wr:.4g} (ncu unit)  SM {d['sm__throughput.avg.pct_of_peak_sustained_elapsed']}%  "
          f"L1 {d['l1tex__throughput.avg.pct_of_peak_sustained_active']}%  L2 {d['lts__throughput.avg.pct_of_peak_sustained_elapsed']}%  "
          f"IPC {d['sm__inst_executed.avg.per_cycle_active']}  warps active {d['sm__warps_active.avg.pct_of_peak_sustained_active']}%  "
          f"inst {d['smsp__inst_executed.sum']}")
    tot = f("smsp__pcsamp_sample_count") or 1.0
    stalls = sorted(((f(f"smsp__pcsamp_warps_issue_stalled_{s}"), s) for s in ST), reverse=True)[:6]
    print("   stalls: " + ", ".join(f"{s} {v / tot * 100:.0f}%" for v, s in stalls))
