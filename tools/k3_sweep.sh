# K3 plan sweep at G = 1: side-chain SMs x small-group threshold (bench value, interleaved twice)
mkdir -p gpurun_out/k3sweep
for rep in 1 2; do
for cfg in deepseek qwen; do
for sg in 12 16 20 28; do
for sm in 128 256; do
  MP_GEMM_SMALL_GRID=$sg MP_GEMM_SPLIT_M=$sm timeout 120 python bench.py --config $cfg --steps 300 --no-cpu-baseline > gpurun_out/k3sweep/$cfg.$sg.$sm.$rep.out 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/k3sweep/$cfg.$sg.$sm.$rep.out') if l.startswith('{')][-1]); print('$cfg sg=$sg split=$sm rep=$rep', round(d['value']/1e6,3), d['clocks']['sm_mhz'])" >> gpurun_out/k3sweep/summary.txt 2>&1
done; done; done; done
