#!/bin/bash
# A/B of the garbling launch: parity subset, headline bench line, and the
# act_kernel<garble> launch's duration / DRAM bytes / instructions under ncu.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/quick_bench.sh
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum \
  --clock-control none -k regex:act_kernel -s 0 -c 1 --csv --log-file gpurun_out/ab_ncu.csv python scripts/ncu_target.py 64 > /dev/null 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/ab_ncu.csv")) if len(r) > 5]
h = rows[0]
for r in rows[1:]:
    print(r[h.index("Metric Name")], r[h.index("Metric Unit")], r[h.index("Metric Value")])
PY
