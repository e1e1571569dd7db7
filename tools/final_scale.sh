# weak-scaling lines as the driver launches them (torchrun, one rank per GPU)
mkdir -p ${OUT:-gpurun_out/final3s}
for N in 2 4; do for c in mixtral deepseek qwen; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29544 \
    bench.py --gpus $N --config $c > ${OUT:-gpurun_out/final3s}/${c}_G$N.json 2> ${OUT:-gpurun_out/final3s}/${c}_G$N.err
  echo "$c G=$N rc=$?" >> ${OUT:-gpurun_out/final3s}/summary.txt
done; done
