# N > 1 plumbing on a one-GPU box: 2 ranks over gloo sharing cuda:0 (replicas cfg2, cfg3 partition,
# reference arm).  Timings are meaningless here; the JSON line and exit codes are what is checked.
export IDK_BENCH_BACKEND=gloo
for c in cfg2 cfg3; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --config $c --steps 3 --warmup 3 --batch 4 > gpurun_out/mr_$c.json 2> gpurun_out/mr_$c.err; echo $c rc=$?
  head -c 400 gpurun_out/mr_$c.json; echo
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo ref rc=$?
head -c 300 gpurun_out/mr_ref.json; echo
