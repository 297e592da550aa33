for shp in "moving 400 250 40000 fsr,ssr" "sensor 1000 1000 20000 fsr"; do
  for v in b4 b4s b2 b4m5 b4m6; do echo "== $v"; SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py $shp; done
done
