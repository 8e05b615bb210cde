# GPU parity suite + smoke only (no bench); outputs under gpurun_out/
timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
