python bench.py --config C1 --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
for lag in 5 10 20 40; do echo "C1 lag_x10=$lag $(LOKI_PIPE_LAG_X10=$lag python tools/one_layer.py --B 1 --S 4096 --reps 20 | tail -1)"; done
for h in 0 1 2; do echo "C1 halves=$h $(LOKI_PIPE_HALVES=$h python tools/one_layer.py --B 1 --S 4096 --reps 20 | tail -1)"; done
for c in 1 2; do echo "C1 ctas/sm=$c $(LOKI_PIPE_CTAS_PER_SM=$c python tools/one_layer.py --B 1 --S 4096 --reps 20 | tail -1)"; done
