# sweep iteration: sweep parity suites, grid timings (digests must not change), ncu at 128 tau
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_reference_cases.py -x -q > gpurun_out/sweep_tests.log 2>&1; echo rc=$? >> gpurun_out/sweep_tests.log
timeout 300 python tools/sweep_ab.py 10 > gpurun_out/ab_v9.jsonl 2> gpurun_out/ab_v9.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cse_tile9 -c 1 -o gpurun_out/cse9_128 -f python tools/cse_probe.py 128 1 1e-14 > gpurun_out/cse9_128.log 2>&1
