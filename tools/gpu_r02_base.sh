set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02/base_c2.json 2> gpurun_out/r02/base_c2.err
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --bins 100 --frames 4096 > gpurun_out/r02/base_b100.json 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --bins 256 --frames 4096 > gpurun_out/r02/base_b256.json 2>&1
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --frames 2048 > gpurun_out/r02/base_c2_2048.json 2>&1
tail -c 600 gpurun_out/r02/base_*.json
