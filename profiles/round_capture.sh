# Round capture on the GPU box: build-matched ncu step profile, bench (both
# arms), launch list.  Outputs in gpurun_out/ (copy the summaries to profiles/).
set -x
for m in fsr ssr; do
  timeout 900 ncu --set full --clock-control none --launch-skip 9 --launch-count 8 \
     -o gpurun_out/step_$m -f python profiles/ncu_step_profile.py run $m > gpurun_out/ncu_step_$m.log 2>&1
done
python profiles/ncu_step_profile.py summarize gpurun_out/step_fsr.ncu-rep gpurun_out/step_ssr.ncu-rep \
   --out gpurun_out/ncu_step.json > /dev/null
cp gpurun_out/ncu_step.json profiles/ncu_step.json
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-long --no-configs \
   > gpurun_out/ncu_launch.log 2>&1
tail -c 1500 gpurun_out/bench.json; echo; cat gpurun_out/bench_ref.json
