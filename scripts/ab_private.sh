cd /root/repo
timeout 400 python -m pytest tests -m gpu -x -q -k "priv or golden or lenet_batch" 2>&1 | tail -1
for lib in "" variants/head.so; do
  DASHGPU_LIB=$lib timeout 300 python bench.py --model lenet5 --private --batch 64 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('[${lib:-in-tree}]', round(d['value'],1), {k:round(v,1) for k,v in d['kernels_ms_per_step'].items()})"
done
