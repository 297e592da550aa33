# build a variant of libspikecam_b200.so with extra nvcc defines: build_variant.sh NAME -DX=Y ...
name=$1; shift
mkdir -p profiles/_ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -static-global-template-stub=false -Iinclude "$@" -o profiles/_ab/lib_$name.so paper_2412_11639_b200/csrc/*.cu
