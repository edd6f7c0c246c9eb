# In-tree build of the B200 library (sm_100a only) and the oracle's C helpers.
NVCC ?= nvcc
NVFLAGS = -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
          -Xcompiler -fPIC -shared
PKG = paper_2506_09594_b200
SRC = $(PKG)/csrc/lrta.cu
HDR = $(wildcard $(PKG)/csrc/*.cuh) include/tenrec_b200.h

all: $(PKG)/libtenrec_b200.so

$(PKG)/libtenrec_b200.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) $(SRC) -o $@

clean:
	rm -f $(PKG)/libtenrec_b200.so

.PHONY: all clean
