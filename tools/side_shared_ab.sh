# fused shared expert rows on the side chain (MP_SIDE_SHARED_ROWS): parity, then interleaved bench A/B
mkdir -p gpurun_out/sshared
for ms in 256 512; do
  MP_SIDE_SHARED_ROWS=$ms timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_layer.py -m gpu -q -x > gpurun_out/sshared/pytest_$ms.log 2>&1
  echo "pytest ms=$ms rc=$? $(tail -1 gpurun_out/sshared/pytest_$ms.log)" >> gpurun_out/sshared/summary.txt
done
for rep in 1 2; do for cfg in deepseek qwen; do for ms in 0 256 512; do for sg in 20 24 28; do
  MP_SIDE_SHARED_ROWS=$ms MP_GEMM_SMALL_GRID=$sg timeout 120 python bench.py --config $cfg --steps 300 --no-cpu-baseline > gpurun_out/sshared/$cfg.$ms.$sg.$rep.out 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/sshared/$cfg.$ms.$sg.$rep.out') if l.startswith('{')][-1]); print('$cfg ms=$ms sg=$sg rep=$rep', round(d['value']/1e6,3), d['clocks']['sm_mhz'], d.get('side_chain_ms'), round(d['stages_ms']['gemm1_swiglu']+d['stages_ms']['gemm2'],4))" >> gpurun_out/sshared/summary.txt 2>&1
done; done; done; done
