for shp in "moving 400 250 40000 ssr" "sensor 1000 1000 20000 ssr" "static 400 250 20000 ssr" "moving 400 250 4000 ssr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
  echo "== sreg"; SPK_PROBE_LIB=profiles/_ab/lib_sreg.so timeout 300 python profiles/phases.py $shp
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_split.py tests/test_time_shards.py -x -q 2>&1 | tail -3
