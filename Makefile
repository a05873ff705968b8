# Builds the B200-native CK-MPM transfer library (sm_100a only) and the
# oracle checker libraries.  `python -c "import __graft_entry__ as g; g.build()"`
# runs this.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -O3 \
          -Xptxas -v,-warn-spills
PKG = paper_2412_10399_b200
SRC = $(PKG)/csrc/ckg_api.cu
HDR = $(wildcard $(PKG)/csrc/*.cuh) include/ckmpm_b200.h

all: $(PKG)/libckmpm_b200.so oracle

$(PKG)/libckmpm_b200.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; false)
	@grep -E "spill|Used" build/ptxas.log | sed -n '1,200p' > build/ptxas_summary.txt || true

oracle:
	$(MAKE) -C oracle all

clean:
	rm -f $(PKG)/libckmpm_b200.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
