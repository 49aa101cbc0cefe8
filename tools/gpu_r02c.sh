mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tc-head" > gpurun_out/r02c_head_tests.log 2>&1; echo rc=$? >> gpurun_out/r02c_head_tests.log
SSJB_HEAD=1 timeout 300 python tools/heavy_phases.py C4 C4_b128 > gpurun_out/r02c_heavy.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_heavy.py -x -q -s > gpurun_out/r02c_heavy_tests.log 2>&1; echo rc=$? >> gpurun_out/r02c_heavy_tests.log
