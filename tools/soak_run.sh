# Soak runs of the NVLink flag protocol at G = 4 (results: gpurun_out/soak/summary.txt).
#   bash tools/soak_run.sh all     tools/soak.py, protocol state checked every 100-200 forwards
#   bash tools/soak_run.sh ev      long chunks with per-forward stage events (bench's timed loop)
#   bash tools/soak_run.sh smi     the soak while nvidia-smi samples every GPU (bench's clock sampler)
#   bash tools/soak_run.sh bench   bench.py's own long timed loops
mkdir -p gpurun_out/soak
run() {  # name, env, script, args...
  name=$1; shift; envs=$1; shift; script=$1; shift
  env $envs timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29511 $script --gpus 4 --warmup 3 "$@" > gpurun_out/soak/$name.out 2> gpurun_out/soak/$name.err
  echo "$name rc=$?" >> gpurun_out/soak/summary.txt
  tail -c 600 gpurun_out/soak/$name.out >> gpurun_out/soak/summary.txt
}
case "${1:-all}" in
  all)
    run ds_a "X=1" tools/soak.py --config deepseek --steps 20000 --chunk=100
    run toy_a "X=1" tools/soak.py --config toy --steps 40000 --chunk=200
    run mix_a "X=1" tools/soak.py --config mixtral --steps 8000 --chunk=100
    run qwen_a "X=1" tools/soak.py --config qwen --steps 20000 --chunk=100
    ;;
  ev)
    run ds_ev "X=1" tools/soak.py --config deepseek --steps 12000 --chunk=3000 --events
    run toy_ev "X=1" tools/soak.py --config toy --steps 40000 --chunk=10000 --events
    ;;
  smi)
    smi_fields=timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active
    for i in 0 1 2 3; do
      nvidia-smi --query-gpu=$smi_fields --format=csv,noheader,nounits -lms 100 -i $i > gpurun_out/soak/smi$i.txt 2>&1 &
    done
    run ds_smi "X=1" tools/soak.py --config deepseek --steps 12000 --chunk=20
    run mix_smi "X=1" tools/soak.py --config mixtral --steps 4000 --chunk=20
    run toy_smi "X=1" tools/soak.py --config toy --steps 20000 --chunk=100
    kill %1 %2 %3 %4
    ;;
  bench)
    run ds_b "X=1" bench.py --config deepseek --steps 3000 --no-cpu-baseline
    run qwen_b "X=1" bench.py --config qwen --steps 3000 --no-cpu-baseline
    run mix_b "X=1" bench.py --config mixtral --steps 1500 --no-cpu-baseline
    run ds_b2 "X=1" bench.py --config deepseek --steps 3000 --no-cpu-baseline
    run mix_b2 "X=1" bench.py --config mixtral --steps 1500 --no-cpu-baseline
    ;;
esac
