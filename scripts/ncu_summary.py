"""Summarise an ncu report: headline metrics, stall reasons, hottest source lines."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed_op_local_ld.sum"]
for r in rows[2:]:
    print("kernel:", r[hdr.index("Kernel Name")][:60])
    for w in want:
        if w in hdr: print(f"  {w} = {r[hdr.index(w)]}")
    vals = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try: vals.append((float(r[i]), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError: pass
    tot = sum(v for v, _ in vals) or 1
    print("  stalls:", ", ".join(f"{n} {100*v/tot:.1f}%" for v, n in sorted(vals, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", "regex:.", "--launch-skip", "0", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
agg = []; cur = None; hdr = None
for r in csv.reader(io.StringIO(src)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name",) or hdr is None and r[0] != "Line No": continue
    if r[0] == "Line No": hdr = r; continue
    try: agg.append((int(r[hdr.index("Warp Stall Sampling (All Samples)")]), int(r[hdr.index("Instructions Executed")]), cur, r[0], r[1][:100]))
    except (ValueError, IndexError, TypeError): pass
ts = sum(a[0] for a in agg) or 1; ti = sum(a[1] for a in agg) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for a in sorted(agg, reverse=True)[:n]:
    print(f"{100*a[0]/ts:5.1f}% smp {100*a[1]/ti:5.1f}% ins  {a[2]}:{a[3]}  {a[4]}")
