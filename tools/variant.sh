#!/bin/bash
# tools/variant.sh NAME "-DFLAG=V ..." : build tools/libmsrep_NAME.so with extra defines (tuning experiments)
name=$1; shift
NCCLH=$(python -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2209_07552_b200/csrc -I$NCCLH/include $*"
nvcc $F -c paper_2209_07552_b200/csrc/kernels.cu -o /tmp/k_$name.o 2>/dev/null && \
nvcc $F -x cu -c paper_2209_07552_b200/csrc/host.cpp -o /tmp/h_$name.o 2>/dev/null && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/libmsrep_$name.so /tmp/k_$name.o /tmp/h_$name.o -L$NCCLH/lib -l:libnccl.so.2 && echo built tools/libmsrep_$name.so
