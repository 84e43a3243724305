# End-of-round ncu evidence for the SMEM-tier kernel (config 2 shape, 1000 MC steps) + launch list
mkdir -p gpurun_out
timeout 600 python bench.py --config 2 --mc-steps 1000 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/c2ncu_plain.json 2>/dev/null; tail -1 gpurun_out/c2ncu_plain.json | head -c 300; echo
timeout 900 ncu --set full --import-source on --clock-control none -k regex:anneal_smem -c 1 -f -o gpurun_out/r02_smem_c2 python bench.py --config 2 --mc-steps 1000 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/c2ncu.log 2>&1; tail -2 gpurun_out/c2ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c2.csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/r02_launches_c2.csv
