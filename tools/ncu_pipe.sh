python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -40 > gpurun_out/pytest_gpu.log
ncu --set full --import-source on --clock-control none -k regex:pipe_decode -c 1 -o gpurun_out/pipe_v2 python tools/one_layer.py --reps 1 > gpurun_out/ncu_pipe.log 2>&1
ncu -i gpurun_out/pipe_v2.ncu-rep --page details --csv > gpurun_out/pipe_v2_details.csv 2>&1
ncu -i gpurun_out/pipe_v2.ncu-rep --page source --csv --print-source cuda > gpurun_out/pipe_v2_source_cuda.csv 2>&1
ncu -i gpurun_out/pipe_v2.ncu-rep --page raw --csv > gpurun_out/pipe_v2_raw.csv 2>&1
