# K3 split plan at G = 1, wider: small-group threshold {256, 384, 512} x side-chain SMs {20, 28, 36}
mkdir -p gpurun_out/k3sweep2
for rep in 1 2; do for cfg in deepseek qwen; do for sm in 256 384 512; do for sg in 20 28 36; do
  MP_GEMM_SMALL_GRID=$sg MP_GEMM_SPLIT_M=$sm timeout 120 python bench.py --config $cfg --steps 300 --no-cpu-baseline > gpurun_out/k3sweep2/$cfg.$sg.$sm.$rep.out 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/k3sweep2/$cfg.$sg.$sm.$rep.out') if l.startswith('{')][-1]); print('$cfg split=$sm sg=$sg rep=$rep', round(d['value']/1e6,3), d['clocks']['sm_mhz'], d.get('side_chain_ms'), round(d['stages_ms']['gemm1_swiglu']+d['stages_ms']['gemm2'],4))" >> gpurun_out/k3sweep2/summary.txt 2>&1
done; done; done; done
