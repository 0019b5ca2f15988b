#!/bin/bash
# tools/variant.sh NAME "-DFLAG=V ..." : a tuning build with extra defines, as a runnable mirror of the repo
# in tools/variants/NAME (symlinks + the variant libmsrep.so in its own package dir).  The product
# binding only ever loads the in-tree paper_2209_07552_b200/libmsrep.so; run a variant with
#   (cd tools/variants/NAME && python bench.py ...)
set -e
name=$1; shift
NCCLH=$(python -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2209_07552_b200/csrc -I$NCCLH/include $*"
nvcc $F -c paper_2209_07552_b200/csrc/kernels.cu -o /tmp/k_$name.o
nvcc $F -c paper_2209_07552_b200/csrc/transpose.cu -o /tmp/t_$name.o
nvcc $F -x cu -c paper_2209_07552_b200/csrc/host.cpp -o /tmp/h_$name.o
d=tools/variants/$name
mkdir -p $d/paper_2209_07552_b200
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/paper_2209_07552_b200/libmsrep.so /tmp/k_$name.o /tmp/t_$name.o /tmp/h_$name.o \
  -L$NCCLH/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCLH/lib
cp paper_2209_07552_b200/__init__.py $d/paper_2209_07552_b200/
for f in bench.py gen oracle tests tools include profiles MEASURED_PEAKS.json __graft_entry__.py pytest.ini; do
  [ -e "$f" ] && ln -sfn "$PWD/$f" "$d/$f"
done
echo "built $d"
