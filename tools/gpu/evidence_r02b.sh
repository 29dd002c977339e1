set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r02b_gpu_tests.log
python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
python tools/sweep_ab.py 20 > gpurun_out/r02b_sweep_grids.jsonl 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02b_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r02b_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:cse_tile9 -c 1 -o gpurun_out/r02b_cse10_32 python tools/cse_probe.py 32 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:cse_tile9 -c 1 -o gpurun_out/r02b_cse10_128 python tools/cse_probe.py 128 1 1e-14 > /dev/null 2>&1
tail -3 gpurun_out/r02b_gpu_tests.log; cat gpurun_out/r02b_sweep_grids.jsonl; head -c 600 gpurun_out/r02b_bench.json
