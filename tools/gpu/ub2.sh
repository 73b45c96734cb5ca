mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_phase_loop.py tests/test_full_size.py -x -q > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
bash tools/gpu/ub.sh
