# round-2 check: full GPU suite, smoke, bench line (ours + reference arm), launch list of the bench, ncu of the sweep tile kernel (32 / 128 tau)
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cse_tile9 -c 1 -o gpurun_out/cse9_32 -f python tools/cse_probe.py 32 1 > gpurun_out/cse9_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cse_tile9 -c 1 -o gpurun_out/cse9_128 -f python tools/cse_probe.py 128 1 1e-14 > gpurun_out/cse9_128.log 2>&1
timeout 600 python tools/sweep_ab.py 10 > gpurun_out/ab_v9.jsonl 2> gpurun_out/ab_v9.err
