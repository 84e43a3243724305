mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/z2_gputests.log 2>&1; tail -3 gpurun_out/z2_gputests.log
python tools/phase_trace.py 12 148 200 > gpurun_out/z2_phase12.txt 2>&1; cat gpurun_out/z2_phase12.txt
python tools/phase_trace.py 8 64 400 > gpurun_out/z2_phase8.txt 2>&1; cat gpurun_out/z2_phase8.txt
