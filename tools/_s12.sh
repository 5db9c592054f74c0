mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  LOKI_TUNING=1 LOKI_SPIN_S=100000 timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"; grep -v "^=========     " gpurun_out/sanitize_$tool.log | tail -6
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'append_kernel|pipe_select' -s 6 -c 2 -o gpurun_out/k0_sel python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-extras --no-parity > gpurun_out/ncu_k0.log 2>&1
ncu -i gpurun_out/k0_sel.ncu-rep --page raw --csv > gpurun_out/k0_sel_raw.csv 2>&1
ncu -i gpurun_out/k0_sel.ncu-rep --page details --csv > gpurun_out/k0_sel_details.csv 2>&1
ls -la gpurun_out/
