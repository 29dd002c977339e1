# A/B: cfg2 sweep with the default library and each build/variants/*.so
# (usage: NTS="32" bash tools/gpu/ab.sh)
shopt -s nullglob
for nt in ${NTS:-32}; do
  python tools/cse_probe.py $nt 8 > gpurun_out/ab_default_$nt.txt 2>&1
  for v in build/variants/*.so; do
    SPG_LIB=$v python tools/cse_probe.py $nt 8 > gpurun_out/ab_$(basename $v .so)_$nt.txt 2>&1
  done
done
