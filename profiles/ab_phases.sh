# A/B: phases of the working tree's library vs another build ($1); extra env via $2
for shp in "moving 400 250 40000 fsr" "sensor 1000 1000 20000 fsr" "static 400 250 20000 fsr"; do
  echo "== new"; env $2 timeout 300 python profiles/phases.py $shp
  echo "== old"; env $2 SPK_PROBE_LIB=$1 timeout 300 python profiles/phases.py $shp
done
