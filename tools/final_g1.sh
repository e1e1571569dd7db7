# round-end style validation on one GPU: smoke, pytest -m gpu, default bench, configs, reference arm
mkdir -p ${OUT:-gpurun_out/final3}
python -c "import __graft_entry__ as g; g.smoke()" > ${OUT:-gpurun_out/final3}/smoke.log 2>&1; echo "smoke rc=$?" >> ${OUT:-gpurun_out/final3}/summary.txt
timeout 1200 python -m pytest tests -m gpu -q -x > ${OUT:-gpurun_out/final3}/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> ${OUT:-gpurun_out/final3}/summary.txt
tail -1 ${OUT:-gpurun_out/final3}/pytest_gpu.log >> ${OUT:-gpurun_out/final3}/summary.txt
timeout 600 python bench.py > ${OUT:-gpurun_out/final3}/bench_default.json 2> ${OUT:-gpurun_out/final3}/bench_default.err; echo "bench default rc=$?" >> ${OUT:-gpurun_out/final3}/summary.txt
for c in deepseek qwen toy; do timeout 300 python bench.py --config $c > ${OUT:-gpurun_out/final3}/bench_$c.json 2> ${OUT:-gpurun_out/final3}/bench_$c.err; echo "bench $c rc=$?" >> ${OUT:-gpurun_out/final3}/summary.txt; done
timeout 600 python bench.py --impl reference > ${OUT:-gpurun_out/final3}/reference.json 2> ${OUT:-gpurun_out/final3}/reference.err; echo "reference rc=$?" >> ${OUT:-gpurun_out/final3}/summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${OUT:-gpurun_out/final3}/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > ${OUT:-gpurun_out/final3}/ncu.log 2>&1; echo "ncu rc=$?" >> ${OUT:-gpurun_out/final3}/summary.txt
