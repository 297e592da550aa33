for pad in 0 4096 14000 32000; do
for shp in "moving 400 250 40000 fsr" "static 400 250 20000 fsr" "sensor 1000 1000 20000 fsr"; do
  echo "== pad $pad"; SPK_K3_PAD=$pad timeout 300 python profiles/phases.py $shp
done
done
echo "== tma"; SPK_TMA=1 timeout 300 python profiles/phases.py moving 400 250 40000 fsr
