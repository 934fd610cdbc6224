# dev: build a PRODUCT-flag variant (no -DKAAS_DEV) of libkaas_b200.so into build/var/<name>.so from the
# current sources with one sed expression applied to one file:
#   bash tools/build_var.sh <name> <file.cu> '<sed expr>'
set -e
name=$1; file=$2; expr=$3
root=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d); mkdir -p $T/p/c $T/include "$root/build/var"
cp "$root"/include/*.h $T/include/
cp "$root"/paper_2212_08146_b200/csrc/*.cu "$root"/paper_2212_08146_b200/csrc/*.cuh $T/p/c/
sed -i "$expr" $T/p/c/$file
cd $T/p/c
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
for f in kaas_abi builtins jacobi cgemm runs; do nvcc $F -c $f.cu -o $f.o 2>/dev/null & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/build/var/$name.so" *.o -lcudart
rm -rf $T
echo "built build/var/$name.so"
