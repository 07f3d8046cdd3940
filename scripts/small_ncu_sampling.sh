timeout 300 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_small -s 5 -c 1 -o gpurun_out/ncu_small_sc3 python scripts/step_graph_time.py 10000 > gpurun_out/ncu_small_sc3.log 2>&1; tail -5 gpurun_out/ncu_small_sc3.log
ncu -i gpurun_out/ncu_small_sc3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_small_sc3_src.csv 2>/dev/null
ncu -i gpurun_out/ncu_small_sc3.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_small_sc3_sass.csv 2>/dev/null
gzip -f gpurun_out/ncu_small_sc3_src.csv gpurun_out/ncu_small_sc3_sass.csv; rm -f gpurun_out/ncu_small_sc3.ncu-rep; ls -la gpurun_out/ncu_small_sc3*
