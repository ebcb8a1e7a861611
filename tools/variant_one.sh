# Build a library variant that differs in ONE source file only: the other objects come from the
# build cache.  bash tools/variant_one.sh <name> <file.cu> [extra nvcc flags]  ->  paper_2005_13471_b200/var/<name>.so
set -e
name=$1; src=$2; shift 2
cs=paper_2005_13471_b200/csrc
mkdir -p paper_2005_13471_b200/var /tmp/var_$name
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude -I$cs "$@" -c $cs/$src -o /tmp/var_$name/${src%.cu}.o
objs=$(ls build/bsct/*.o | grep -v "/${src%.cu}-")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2005_13471_b200/var/$name.so \
  /tmp/var_$name/${src%.cu}.o $objs -lcudart_static -lrt -ldl -lpthread
echo paper_2005_13471_b200/var/$name.so
