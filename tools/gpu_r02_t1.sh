# r02: full -m gpu suite on the stripped library + first bench lines
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02/pytest_gpu_t1.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/r02/pytest_gpu_t1.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/t1_c2.json 2> gpurun_out/r02/t1_c2.err
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --bins 100 --frames 4096 > gpurun_out/r02/t1_b100.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --bins 256 --frames 4096 > gpurun_out/r02/t1_b256.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --config C4 > gpurun_out/r02/t1_c4.json 2>&1
for f in gpurun_out/r02/t1_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['roofline']['achieved']), d['ms_per_step'])" ; done
