for shp in "sensor 1000 1000 20000 ssr" "moving 400 250 40000 ssr" "moving 400 250 4000 ssr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
  for v in d7 d10 d12 d16; do echo "== $v"; SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py $shp; done
done
