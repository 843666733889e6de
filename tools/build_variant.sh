# Build an A/B variant of the library with extra nvcc defines:  bash tools/build_variant.sh <name> <file.cu> -DX=1 ...
set -e
name=$1; src=$2; shift 2
mkdir -p ab/obj_$name
for f in build/*.o; do cp $f ab/obj_$name/; done
base=$(basename $src .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude "$@" -c $src -o ab/obj_$name/$base.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/lib_$name.so ab/obj_$name/*.o
echo built ab/lib_$name.so
