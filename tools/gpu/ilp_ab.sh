# sweep S-loop ILP A/B: default library (2 evaluations in flight per lane) vs build/variants ilp3 / ilp4; bits must match
set -x
timeout 300 python tools/sweep_ab.py 10 > gpurun_out/ilp2.jsonl 2> gpurun_out/ilp2.err
SPG_LIB=build/variants/ilp3.so timeout 300 python tools/sweep_ab.py 10 > gpurun_out/ilp3.jsonl 2> gpurun_out/ilp3.err
SPG_LIB=build/variants/ilp4.so timeout 300 python tools/sweep_ab.py 10 > gpurun_out/ilp4.jsonl 2> gpurun_out/ilp4.err
SPG_CSE_FOLD=2 timeout 300 python tools/sweep_ab.py 10 > gpurun_out/fold2.jsonl 2> gpurun_out/fold2.err
