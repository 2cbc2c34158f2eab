"""Aggregate an ncu source page (instructions / stall samples) per function of dash_device.cuh."""
import bisect, csv, io, re, subprocess, sys
rep = sys.argv[1]
fn_file = "paper_2302_06361_b200/csrc/dash_device.cuh"
funcs = []
for i, line in enumerate(open(fn_file), 1):
    m = re.match(r"^(DASH_HD|template|__device__|static inline|struct)\s.*?(\w+)\s*\(", line)
    if m: funcs.append((i, m.group(2)))
starts = [f[0] for f in funcs]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", "regex:.",
                      "--launch-skip", sys.argv[2] if len(sys.argv) > 2 else "0", "--launch-count", "1"], capture_output=True, text=True).stdout
cur = None; hdr = None; agg = {}
for r in csv.reader(io.StringIO(src)):
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or not r[0]: continue
    try:
        ln = int(r[0]); ins = int(r[hdr.index("Instructions Executed")]); smp = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    if cur == "dash_device.cuh":
        i = bisect.bisect_right(starts, ln) - 1
        key = funcs[i][1] if i >= 0 else "?"
    else:
        key = cur
    a = agg.setdefault(key, [0, 0]); a[0] += ins; a[1] += smp
ti = sum(v[0] for v in agg.values()) or 1; ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {ti:.3e}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{100*v[0]/ti:5.1f}% ins {100*v[1]/ts:5.1f}% smp  {k}")
