# K2 / K5 column slices A/B at G = 1 (bench stages and value, interleaved twice)
mkdir -p gpurun_out/slices
MP_COMBINE_SLICES=2 MP_PERMUTE_SLICES=8 timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/slices/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/slices/summary.txt; tail -1 gpurun_out/slices/pytest.log >> gpurun_out/slices/summary.txt
for rep in 1 2; do for cfg in deepseek mixtral; do for v in "0 1" "8 1" "0 2" "8 2" "16 4"; do
  set -- $v
  if [ "$1" = "0" ]; then PS=""; else PS="MP_PERMUTE_SLICES=$1"; fi
  env $PS MP_COMBINE_SLICES=$2 timeout 120 python bench.py --config $cfg --steps 300 --no-cpu-baseline > gpurun_out/slices/$cfg.$1.$2.$rep.out 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/slices/$cfg.$1.$2.$rep.out') if l.startswith('{')][-1]); s=d['stages_ms']; print('$cfg perm=$1 comb=$2 rep=$rep', round(d['value']/1e6,3), d['clocks']['sm_mhz'], 'permute', round(s['permute_dispatch']*1e3,1), 'combine', round(s['combine_return']*1e3,1))" >> gpurun_out/slices/summary.txt 2>&1
done; done; done
