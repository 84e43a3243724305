cd paper_2203_09353_b200 && cp libtaskgemm_b200.so new_taskgemm.so && cp old_taskgemm.so libtaskgemm_b200.so && cd ..
echo "== old"; bash tools/gpu_runs/_gpu_r02sturm.sh 2>&1 | grep -v pytest | head -3
cd paper_2203_09353_b200 && cp new_taskgemm.so libtaskgemm_b200.so && cd ..
echo "== new"; bash tools/gpu_runs/_gpu_r02sturm.sh
