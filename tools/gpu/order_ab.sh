# CTA-order A/B for the leaf GEMM: L=32 and L=64 config-5 products (tools/profile_leaf.py),
# SPG_ORDER 1 = row-major, 2+s = strips of 2^s rows
for L in ${LS:-32 64}; do for o in ${ORDERS:-1 4 5 6}; do
  echo "L=$L order=$o $(SPG_ORDER=$o python tools/profile_leaf.py $L 2>&1 | tail -1)" >> gpurun_out/order_ab.txt
done; done
