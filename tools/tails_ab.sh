# pair-tile tails on the side chain (MP_GEMM_TAILS): parity first, then interleaved bench A/B
mkdir -p gpurun_out/tails
MP_GEMM_TAILS=128 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_layer.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/tails/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/tails/summary.txt; tail -2 gpurun_out/tails/pytest.log >> gpurun_out/tails/summary.txt
for rep in 1 2; do for cfg in deepseek qwen; do for t in 0 128 64; do for sg in 20 24; do
  MP_GEMM_TAILS=$t MP_GEMM_SMALL_GRID=$sg timeout 120 python bench.py --config $cfg --steps 300 --no-cpu-baseline > gpurun_out/tails/$cfg.$t.$sg.$rep.out 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/tails/$cfg.$t.$sg.$rep.out') if l.startswith('{')][-1]); print('$cfg tails=$t sg=$sg rep=$rep', round(d['value']/1e6,3), d['clocks']['sm_mhz'], d.get('side_chain_ms'), round(d['stages_ms']['gemm1_swiglu']+d['stages_ms']['gemm2'],4))" >> gpurun_out/tails/summary.txt 2>&1
done; done; done; done
