# sweep iteration: sweep parity suites + the large pins, grid timings (digests must not change)
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py tests/test_gpu_reference_cases.py tests/test_gpu_pins.py tests/test_distributed_panels.py -x -q --durations=8 > gpurun_out/sweep_tests.log 2>&1; echo rc=$? >> gpurun_out/sweep_tests.log
timeout 300 python tools/sweep_ab.py 10 > gpurun_out/ab_v9.jsonl 2> gpurun_out/ab_v9.err
SPG_TRACE=1 timeout 600 python -c "
import sys; sys.path.insert(0, 'tests')
from large_cases import GpuCase
from paper_2005_10680_b200 import _native as nat
import time
ctx = nat.Context(0)
g = GpuCase(ctx, 'cfg5-L32')
for _ in range(2):
    t0 = time.perf_counter(); b = nat.cse(ctx, g.A_norms, g.B_norms, g.taus); print('cfg5-L32 one-GPU sweep s', round(time.perf_counter() - t0, 3), flush=True)
" > gpurun_out/cfg5_l32_sweep.log 2>&1
