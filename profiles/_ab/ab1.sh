for v in base w11 w7 w5; do
  echo "== $v"
  SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py moving 400 250 40000 fsr,ssr
  SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py sensor 1000 1000 20000 fsr
  SPK_PROBE_LIB=profiles/_ab/lib_$v.so timeout 300 python profiles/phases.py static 400 250 20000 fsr
done
