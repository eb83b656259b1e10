mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "wide or locality or residency or pool_grows or multi_device or batch_stream" 2>&1 | tail -4
timeout 300 python scripts/prof_run.py --config 5 --scale 1.0 --runs 3
timeout 300 python scripts/prof_run.py --config 5 --scale 1.0 --runs 3 --shard 0/8
timeout 300 python scripts/prof_run.py --config 4 --scale 0.1 --runs 3 --flags 0
XB_BENCH_FUNCTIONAL=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_n2_functional.json 2> gpurun_out/bench_n2_functional.err; echo "n2 rc=$?"; tail -c 1500 gpurun_out/bench_n2_functional.json
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
