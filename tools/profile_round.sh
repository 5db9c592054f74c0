# Measurement recipe behind profiles/ (run on a B200 via gpurun; outputs in gpurun_out/):
#   GPU tests, bench lines (C2 headline, TGT north-star shape, GQA C3 / C4 / C5s, C1), ncu launch lists with
#   DRAM bytes per launch (-> profiles/roofline_traffic.json via tools/traffic_from_launches.py), and one
#   ncu --set full capture of a layer's pipe launches (split layers: the A-only and the B-only launch).
set -x
timeout 900 python -m pytest tests -m gpu -q --tb=short > gpurun_out/tests_gpu.log 2>&1
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config TGT --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_tgt.json 2> gpurun_out/bench_tgt.err
python bench.py --config C1 --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config C3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config C5s --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5s.json 2> gpurun_out/bench_c5s.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'pipe_decode|append_kernel' -c 192 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'pipe_decode|append_kernel' -c 60 --csv --log-file gpurun_out/launches_tgt.csv \
    python bench.py --config TGT --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:pipe_decode -s 40 -c 2 -o gpurun_out/pipe_c2 \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/pipe_c2.ncu-rep --page raw --csv > gpurun_out/pipe_c2_raw.csv 2>&1
