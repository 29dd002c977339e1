# A/B of build/variants/*.so on the config-5-style leaf GEMMs (tools/profile_leaf.py L)
for L in ${LS:-32 64}; do
  echo "default L=$L $(python tools/profile_leaf.py $L 2>&1 | tail -1)" >> gpurun_out/gemm_ab.txt
  for v in build/variants/*.so; do
    echo "$(basename $v .so) L=$L $(SPG_LIB=$v python tools/profile_leaf.py $L 2>&1 | tail -1)" >> gpurun_out/gemm_ab.txt
  done
done
