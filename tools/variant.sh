# Build a library variant with one source recompiled under extra -D flags:
#   bash tools/variant.sh NAME SOURCE.cu -DFOO=1 ...  ->  paper_2005_13471_b200/var/NAME.so
# (time it with BSCT_LIB=paper_2005_13471_b200/var/NAME.so; the var/ dir is git-ignored)
set -e
name=$1; src=$2; shift 2
python -m paper_2005_13471_b200.build > /dev/null
mkdir -p paper_2005_13471_b200/var /tmp/bsct_var
objs=$(python - "$src" <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2005_13471_b200 import build as b
hh = b._header_hash()
print(" ".join(b._obj_path(s, hh) for s in b._sources() if s != sys.argv[1]))
PY
)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Xptxas -warn-spills -Iinclude -Ipaper_2005_13471_b200/csrc "$@" -c paper_2005_13471_b200/csrc/$src -o /tmp/bsct_var/$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2005_13471_b200/var/$name.so $objs /tmp/bsct_var/$name.o \
  -lcudart_static -lrt -ldl -lpthread
echo paper_2005_13471_b200/var/$name.so
