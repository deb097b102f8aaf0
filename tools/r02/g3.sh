mkdir -p gpurun_out
HC_SHARD_ALPHA=12.7 timeout -s KILL 900 python tools/shard_times.py 20 22 > gpurun_out/g3_shards_a127.txt 2>&1; tail -8 gpurun_out/g3_shards_a127.txt
