# multi-GPU randomised parity fuzz (tests/mgpu_worker.py random cases, every row vs the oracle)
mkdir -p gpurun_out/fuzz
for G in 4 3 2; do
  MGPU_CASES=rand MGPU_RAND_SEEDS=$1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $G \
    --master-addr 127.0.0.1 --master-port 29581 tests/mgpu_worker.py > gpurun_out/fuzz/G$G.out 2> gpurun_out/fuzz/G$G.err
  echo "G=$G rc=$? $(grep -h 'mgpu ok' gpurun_out/fuzz/G$G.out)" >> gpurun_out/fuzz/summary.txt
done
