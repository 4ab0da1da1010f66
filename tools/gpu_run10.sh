mkdir -p gpurun_out/s11
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s11/pytest.log 2>&1; tail -5 gpurun_out/s11/pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/s11/smoke.log 2>&1; tail -3 gpurun_out/s11/smoke.log
