for shp in "sensor 1000 1000 20000 ssr" "moving 400 250 40000 ssr" "static 400 250 20000 ssr" "range 400 250 100000 ssr" "moving 400 250 4000 ssr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
  echo "== prev"; SPK_PROBE_LIB=profiles/_ab/lib_prev.so timeout 300 python profiles/phases.py $shp
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
