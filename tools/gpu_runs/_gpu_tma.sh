mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in 3 4; do timeout 400 python bench.py --config $c --steps 2 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -c 400 gpurun_out/bench_c$c.json; echo; done
timeout 300 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 300 gpurun_out/bench_c5.json; echo
for c in 3 4; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:anneal_hbm_kernel -c 1 -f -o gpurun_out/hbm_tma_c$c python bench.py --config $c --mc-steps 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c$c.log 2>&1; tail -2 gpurun_out/ncu_c$c.log
done
