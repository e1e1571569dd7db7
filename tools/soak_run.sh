# soak runs of the flag protocol at G = 4 (tools/soak.py; bench.py timed loops)
mkdir -p gpurun_out/soak
run() {  # name, env, script args...
  name=$1; shift; envs=$1; shift; script=$1; shift
  env $envs timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29511 $script --gpus 4 --warmup 3 "$@" > gpurun_out/soak/$name.out 2> gpurun_out/soak/$name.err
  echo "$name rc=$?" >> gpurun_out/soak/summary.txt
  tail -c 600 gpurun_out/soak/$name.out >> gpurun_out/soak/summary.txt
}
case "${1:-all}" in
  ev)
    run ds_ev "X=1" tools/soak.py --config deepseek --steps 12000 --chunk=3000 --events
    run toy_ev "X=1" tools/soak.py --config toy --steps 40000 --chunk=10000 --events
    run ds_bench "X=1" bench.py --config deepseek --steps 3000 --no-cpu-baseline
    run ds_bench_nopdl "MP_ROUTER_PDL=0" bench.py --config deepseek --steps 3000 --no-cpu-baseline
    ;;
  all)
    run ds_a "X=1" tools/soak.py --config deepseek --steps 20000 --chunk=100
    run toy_a "X=1" tools/soak.py --config toy --steps 40000 --chunk=200
    run mix_a "X=1" tools/soak.py --config mixtral --steps 8000 --chunk=100
    run qwen_a "X=1" tools/soak.py --config qwen --steps 20000 --chunk=100
    ;;
esac
if [ "${1:-}" = "pdl" ]; then
  run ds_nopdl1 "MP_ROUTER_PDL=0" bench.py --config deepseek --steps 3000 --no-cpu-baseline
  run toy_nopdl "MP_ROUTER_PDL=0" bench.py --config toy --steps 20000 --no-cpu-baseline
  run ds_pdl_noclk "MP_BENCH_NO_CLOCKS=1" bench.py --config deepseek --steps 3000 --no-cpu-baseline
  run ds_nopdl2 "MP_ROUTER_PDL=0" bench.py --config deepseek --steps 3000 --no-cpu-baseline
fi
if [ "${1:-}" = "confirm" ]; then
  run ds_c1 "X=1" bench.py --config deepseek --steps 3000 --no-cpu-baseline
  run qwen_c1 "X=1" bench.py --config qwen --steps 3000 --no-cpu-baseline
  run mix_c1 "X=1" bench.py --config mixtral --steps 1500 --no-cpu-baseline
  run ds_c2 "X=1" bench.py --config deepseek --steps 3000 --no-cpu-baseline
  for v in 0 1 0 1; do
    CUDA_VISIBLE_DEVICES=0 MP_ROUTER_PDL=$v timeout 200 python bench.py --no-cpu-baseline > gpurun_out/soak/g1_mix_pdl$v.out 2>&1
    echo "g1 mixtral pdl=$v rc=$?" >> gpurun_out/soak/summary.txt
    python -c "import json,sys; d=json.loads([l for l in open('gpurun_out/soak/g1_mix_pdl$v.out') if l.startswith('{')][-1]); print(d['value'], d['ms_per_step'], d['clocks'])" >> gpurun_out/soak/summary.txt 2>&1
  done
fi
if [ "${1:-}" = "smi" ]; then
  # the soak under bench.py's clock sampler (nvidia-smi -lms 100 on every GPU)
  for i in 0 1 2 3; do nvidia-smi --query-gpu=timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits -lms 100 -i $i > gpurun_out/soak/smi$i.txt 2>&1 & done
  run ds_smi "X=1" tools/soak.py --config deepseek --steps 12000 --chunk=20
  run mix_smi "X=1" tools/soak.py --config mixtral --steps 4000 --chunk=20
  run toy_smi "X=1" tools/soak.py --config toy --steps 20000 --chunk=100
  kill %1 %2 %3 %4
fi
if [ "${1:-}" = "bench" ]; then
  # bench.py's own long timed loops at G = 4 (settle / e2e loop counts agreed over the ranks)
  run ds_b "X=1" bench.py --config deepseek --steps 3000 --no-cpu-baseline
  run qwen_b "X=1" bench.py --config qwen --steps 3000 --no-cpu-baseline
  run mix_b "X=1" bench.py --config mixtral --steps 1500 --no-cpu-baseline
  run ds_b2 "X=1" bench.py --config deepseek --steps 3000 --no-cpu-baseline
  run mix_b2 "X=1" bench.py --config mixtral --steps 1500 --no-cpu-baseline
fi
