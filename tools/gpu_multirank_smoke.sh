# Smoke test of bench.py's multi-rank path on ONE GPU with host-side (gloo)
# collectives: 2 ranks share the device, no kernel waits on another rank.
# Exercises the camera-block shards, the batched track-list gather and the
# rank-0 shard_check against a single-process run.
mkdir -p gpurun_out
CFG=${1:-c5}
V2D_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 20 --warmup 3 \
  --config $CFG --no-cpu-baseline > gpurun_out/multirank_$CFG.log 2>&1; echo multirank_$CFG=$?
grep "^{" gpurun_out/multirank_$CFG.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'shard_check', d.get('shard_check'), 'collectives', d.get('collectives'))" 2>&1 | cut -c1-600
tail -3 gpurun_out/multirank_$CFG.log | cut -c1-300
