for shp in "moving 400 250 40000 fsr,ssr" "sensor 1000 1000 20000 fsr,ssr" "static 400 250 20000 fsr,ssr" "moving 400 250 4000 fsr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
done
python -m pytest tests/test_gpu_parity.py tests/test_split.py tests/test_limits.py -x -q 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_segment" --launch-skip 2 --launch-count 1 -o gpurun_out/k2_fsr -f python profiles/one_recon.py moving 400 250 40000 fsr 3 > gpurun_out/ncu_k2.log 2>&1; tail -2 gpurun_out/ncu_k2.log
