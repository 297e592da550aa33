for shp in "sensor 1000 1000 20000 ssr" "moving 400 250 40000 ssr" "static 400 250 20000 ssr" "range 400 250 100000 ssr" "static 400 250 4000 ssr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
  for v in r1 r2 r4; do echo "== $v"; SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py $shp; done
done
