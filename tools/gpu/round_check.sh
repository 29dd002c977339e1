# full GPU suite, bench line, ncu capture of the sweep tile kernel, launch list of one sweep
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash tools/gpu/cse_ncu.sh 8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/cse_probe.py 32 2 > gpurun_out/cse_launches.csv 2>&1
