# full ncu capture of the cfg2 leaf GEMM launch (source-level shared-memory wavefront attribution)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:leaf_gemm_dmma -c 1 -o gpurun_out/gemm_full -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/gemm_ncu.log 2>&1
