mkdir -p gpurun_out
export TG_HBM_QUEUE=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:anneal_queue -c 1 -o gpurun_out/c_q20 -f python tools/prof_hbm_run.py 20 64 3 > gpurun_out/c_q20.log 2>&1; tail -2 gpurun_out/c_q20.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:anneal_queue -c 1 -o gpurun_out/c_q14 -f python tools/prof_hbm_run.py 14 256 20 > gpurun_out/c_q14.log 2>&1; tail -2 gpurun_out/c_q14.log
export TG_HBM_QUEUE=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:anneal_hbm -c 1 -o gpurun_out/c_c14 -f python tools/prof_hbm_run.py 14 256 20 > gpurun_out/c_c14.log 2>&1; tail -2 gpurun_out/c_c14.log
python tools/prof_hbm_run.py 14 256 20; TG_HBM_QUEUE=1 python tools/prof_hbm_run.py 14 256 20
