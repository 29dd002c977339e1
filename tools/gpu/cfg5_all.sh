# config 5 at full size, every rank of 8 in turn, leaf sizes 128/64/32, three deltas each
for L in 128 64 32; do
  timeout 1500 python tools/cfg4_shard.py --config 5 --leaf $L --all-ranks >> gpurun_out/cfg5_all.jsonl 2>> gpurun_out/cfg5_all.err
done
