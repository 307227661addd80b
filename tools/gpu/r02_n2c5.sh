# config 5 split over 2 ranks sharing the box's one GPU (gloo halo): the Kuhn slab path at full size
mkdir -p gpurun_out
FPB_DIST_BACKEND=gloo timeout 1200 python bench.py --gpus 2 --steps 5 --warmup 3 --e2e-steps 0 --soak 0 --no-configs --no-cpu-baseline > gpurun_out/bench_n2c5.json 2> gpurun_out/bench_n2c5.err; head -c 300 gpurun_out/bench_n2c5.json; echo; python -c "import json;d=json.load(open('gpurun_out/bench_n2c5.json'));print(d.get('multi_gpu'),d.get('phases'),d.get('gpu_launches'),d.get('kernels_ms'));print(json.dumps(d.get('dist_solver'))[:400])"; tail -3 gpurun_out/bench_n2c5.err
