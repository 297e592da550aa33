# phases of several library builds on one scene: ab_multi.sh "SCENE W H T M" lib1 lib2 ...
shp=$1; shift
echo "== tree"; timeout 300 python profiles/phases.py $shp
for l in "$@"; do echo "== $l"; SPK_PROBE_LIB=$l timeout 300 python profiles/phases.py $shp; done
