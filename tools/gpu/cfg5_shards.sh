# config 5 at full size (N = 131072), rank 0 of 8, leaf sizes 32/64/128, three deltas each
for L in 128 64 32; do
  timeout 900 python tools/cfg4_shard.py --config 5 --leaf $L >> gpurun_out/cfg5_shards.jsonl 2>> gpurun_out/cfg5_shards.err
done
