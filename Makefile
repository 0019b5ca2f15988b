# Native build: libmsrep.so (product, sm_100a), liboracle.so (test oracle), libgen.so (inputs).
PY        ?= python
NCCL_HOME := $(shell $(PY) -c "import nvidia.nccl as m; print(list(m.__path__)[0])")
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -v \
             -Iinclude -Ipaper_2209_07552_b200/csrc -I$(NCCL_HOME)/include
PKG       := paper_2209_07552_b200
SRCS      := $(PKG)/csrc/kernels.cu $(PKG)/csrc/transpose.cu $(PKG)/csrc/host.cpp
HDRS      := include/msrep.h $(PKG)/csrc/internal.h

all: $(PKG)/libmsrep.so oracle/liboracle.so gen/libgen.so

$(PKG)/build/kernels.o: $(PKG)/csrc/kernels.cu $(HDRS)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(PKG)/build/ptxas.log || (cat $(PKG)/build/ptxas.log; false)

$(PKG)/build/transpose.o: $(PKG)/csrc/transpose.cu $(HDRS)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(PKG)/build/ptxas_transpose.log || (cat $(PKG)/build/ptxas_transpose.log; false)

$(PKG)/build/host.o: $(PKG)/csrc/host.cpp $(HDRS)
	@mkdir -p $(PKG)/build
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(PKG)/libmsrep.so: $(PKG)/build/kernels.o $(PKG)/build/transpose.o $(PKG)/build/host.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -L$(NCCL_HOME)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_HOME)/lib

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -std=c99 -ffp-contract=off -fno-fast-math -fPIC -shared -o $@ $< -lm

gen/libgen.so: gen/gen.cpp
	g++ -O2 -std=c++17 -fPIC -shared -pthread -o $@ $<

clean:
	rm -rf $(PKG)/build $(PKG)/libmsrep.so oracle/liboracle.so gen/libgen.so

.PHONY: all clean
