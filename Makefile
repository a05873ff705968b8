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

all: $(PKG)/libckmpm_b200.so oracle dropin

$(PKG)/libckmpm_b200.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build/ptxas.log || (cat build/ptxas.log; false)
	@grep -E "spill|Used" build/ptxas.log | sed -n '1,200p' > build/ptxas_summary.txt || true

oracle:
	$(MAKE) -C oracle all

clean:
	rm -f $(PKG)/libckmpm_b200.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean

# C++ drop-in test binary (needs the reference headers; built where they exist,
# the binary travels to the GPU box).
REF ?= /root/reference
# nlohmann/json for the reference's io.hpp (file-format comparison in the io test)
JSON_DIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
JSON_INC = $(if $(wildcard $(JSON_DIR)/json.hpp),-I$(JSON_DIR),)
DROPIN_BIN = tests/cpp/_bin/dropin_test
dropin: $(PKG)/libckmpm_b200.so
	@if [ -d $(REF)/proj/include/ckmpm ]; then \
	  mkdir -p tests/cpp/_bin && g++ -std=gnu++20 -O3 -DNDEBUG -fno-math-errno -pthread \
	    -I$(REF)/proj/include -Iinclude $(JSON_INC) tests/cpp/dropin_test.cpp -L$(PKG) -lckmpm_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../../$(PKG)' -o $(DROPIN_BIN) ; \
	else echo "reference tree absent: keeping prebuilt $(DROPIN_BIN)"; fi

.PHONY: dropin
