for shp in "moving 400 250 40000 ssr" "moving 400 250 4000 ssr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
  echo "== smem2"; SPK_PROBE_LIB=profiles/_ab/lib_smem2.so timeout 300 python profiles/phases.py $shp
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
