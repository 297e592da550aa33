for shp in "sensor 1000 1000 20000 ssr" "moving 400 250 40000 ssr" "static 400 250 20000 ssr" "range 400 250 100000 ssr"; do
  for v in u8 u1 u2 u1r1 u1r2; do echo "== $v"; SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py $shp; done
done
