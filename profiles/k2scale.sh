set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for shp in "400 250 40000" "400 125 40000" "400 64 40000" "400 500 40000" "400 250 20000" "400 1000 40000"; do
  timeout 300 python profiles/phases.py moving $shp fsr
done
timeout 300 python profiles/phases.py moving 400 250 40000 ssr
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_s1.json 2> gpurun_out/bench_s1.err
tail -c 3000 gpurun_out/bench_s1.json
