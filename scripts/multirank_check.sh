# functional multi-rank check on one GPU (gloo, ranks share cuda:0)
export SPMESL_BENCH_SHARE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr2.json 2> gpurun_out/mr2.err; echo "torchrun rc=$?"
tail -3 gpurun_out/mr2.err; cat gpurun_out/mr2.json | cut -c1-400
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"; cat gpurun_out/ref.json | cut -c1-300
