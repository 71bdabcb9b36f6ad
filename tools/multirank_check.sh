# Plumbing of the N>1 bench path on a one-GPU box: 2 ranks share cuda:0 over
# gloo (nothing waits on another rank's kernels); real runs: one GPU per rank, NCCL.
O=gpurun_out
export HOGB200_BENCH_SAME_GPU=1 HOGB200_BENCH_BACKEND=gloo
for c in c2 c4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus 2 --config $c --steps 5 --warmup 3 > $O/mr_$c.json 2> $O/mr_$c.err
  echo "$c rc=$? lines=$(grep -c metric $O/mr_$c.json)"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > $O/mr_ref.json 2> $O/mr_ref.err
echo "ref rc=$? lines=$(grep -c metric $O/mr_ref.json)"
