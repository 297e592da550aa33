for shp in "moving 400 250 40000 fsr" "sensor 1000 1000 20000 fsr,ssr" "static 400 250 20000 fsr,ssr" "range 400 250 200000 fsr"; do
  echo "== new"; timeout 300 python profiles/phases.py $shp
  for v in pl fo plfo; do echo "== $v"; SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py $shp; done
done
