# Measurement recipe behind profiles/ (run on a B200 via gpurun; outputs in gpurun_out/):
#   bench lines (C2 headline, TGT north-star shape, GQA C3 / C4), ncu launch lists with DRAM bytes
#   per launch (profiles/roofline_traffic.json), and one ncu --set full capture of the pipe kernel.
set -x
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config TGT --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_tgt.json 2> gpurun_out/bench_tgt.err
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'pipe_decode|append_kernel' -c 128 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'pipe_decode|append_kernel' -c 40 --csv --log-file gpurun_out/launches_tgt.csv \
    python bench.py --config TGT --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:pipe_decode -s 40 -c 1 -o gpurun_out/pipe_c2 \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/pipe_c2.ncu-rep --page raw --csv > gpurun_out/pipe_c2_raw.csv 2>&1
