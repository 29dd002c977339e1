# K5 CTA order A/B on cfg2: row-major (1) vs strips of 2 / 4 block rows (3 / 4): bench value and ncu DRAM traffic of the GEMM
set -x
for O in 1 3 4; do
  SPG_ORDER=$O timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/order_$O.json 2> gpurun_out/order_$O.err
done
for O in 1 3 4; do
  SPG_ORDER=$O timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:leaf_gemm -c 1 --csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/order_ncu_$O.csv 2> gpurun_out/order_ncu_$O.err
done
