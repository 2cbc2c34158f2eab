for v in libV0 libV1 libV2 lib_01e6910 lib_d29ad2a; do
  for m in "model_a --batch 1 --steps 100 --warmup 10" "model_a --batch 64 --steps 20 --warmup 3"; do
    DASHGPU_LIB=variants/$v.so python bench.py --model $m --k 8 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v', '$m'.split()[2], round(d['value'],1),{k:round(v,3) for k,v in d['kernels_ms_per_step'].items() if k.startswith('act')})"
  done
done
