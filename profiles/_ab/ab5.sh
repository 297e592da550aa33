for shp in "moving 400 250 40000 fsr" "sensor 1000 1000 20000 fsr"; do
  for v in b4 e1 e2 e3; do echo "== $v"; SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py $shp; done
done
