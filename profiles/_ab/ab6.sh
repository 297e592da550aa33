for shp in "moving 400 250 40000 fsr,ssr" "sensor 1000 1000 20000 fsr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
  for v in b4 pb8 pb2 ps32 ps128 pm3 pm5; do echo "== $v"; SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py $shp; done
done
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
