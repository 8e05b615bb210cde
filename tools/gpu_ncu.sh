# one ncu --set full capture of the current top kernels (run plain first)
timeout 300 python tools/run_layer.py stem7x7 c2_1x1_64_256 c3_1x1_256_128 --iters 2 --batch 256 > gpurun_out/run_layer.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"conv_(tc|ws)_kernel" -c 6 \
  -o gpurun_out/prof_r01d python tools/run_layer.py stem7x7 c2_1x1_64_256 c3_1x1_256_128 --iters 2 --batch 256 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log; ls -la gpurun_out/prof_r01d.ncu-rep
