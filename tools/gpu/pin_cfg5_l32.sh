# reference pin of BASELINE config 5 at L = 32 (full size): GPU side + oracle/_ref on the box's host cores; fixture copied back
set -x
timeout 4500 python tests/golden/make_large_pins.py cfg5-L32 > gpurun_out/pin_cfg5_l32.log 2>&1; echo rc=$? >> gpurun_out/pin_cfg5_l32.log
cp tests/golden/large/cfg5-L32.json tests/golden/large/cfg5-L32.npz gpurun_out/ 2>/dev/null
nproc >> gpurun_out/pin_cfg5_l32.log
