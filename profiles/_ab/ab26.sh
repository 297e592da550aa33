for shp in "moving 400 250 40000 fsr,ssr" "sensor 1000 1000 20000 fsr" "static 400 250 20000 fsr" "moving 400 250 4000 fsr" "static 400 250 4000 fsr" "range 400 250 200000 fsr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
  echo "== prev"; SPK_PROBE_LIB=profiles/_ab/lib_prev.so timeout 300 python profiles/phases.py $shp
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_split.py tests/test_time_shards.py tests/test_limits.py -x -q 2>&1 | tail -3
