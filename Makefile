# Build of the B200-native FastNN-Lite path (sm_100a only) and its CPU checkers.
#
#   paper_2503_10017_b200/libfastnn_b200.so  C-ABI + CUDA kernels (include/fastnn_b200.h)
#   paper_2503_10017_b200/libfastnn.so       drop-in C++ API (include/fastnn/*.hpp)
#   paper_2503_10017_b200/_fastnn*.so        drop-in Python surface
#   oracle/_ref/...                          test-only checkers (oracle/Makefile)
#
# Everything is built in-tree so the .so files travel with the repo snapshot.

PY      ?= python3
PKG     := paper_2503_10017_b200
CSRC    := $(PKG)/csrc
NVCC    ?= nvcc
EXT     := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
PYINC   := $(shell $(PY) -c "import sysconfig;print(sysconfig.get_paths()['include'])")
PYBIND  := $(shell $(PY) -c "import pybind11;print(pybind11.get_include())")
JSONDIR ?= $(shell $(PY) -c "import os,site;c=[os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann') for p in site.getsitepackages()];print(next(x for x in c if os.path.exists(x)))")
CUTLASS ?= $(shell $(PY) -c "import os,site;c=[os.path.join(p,'flashinfer/data/cutlass/include') for p in site.getsitepackages()];print(next((x for x in c if os.path.exists(x)),''))")

ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -std=c++17 -O3 -lineinfo --fmad=false -Xcompiler -fPIC -Iinclude -I$(CSRC) \
           --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS:= -std=c++20 -O2 -march=x86-64-v3 -ffp-contract=off -fPIC -Wall -Iinclude -I$(CSRC)/host -I$(JSONDIR)

CU_SRC  := $(CSRC)/capi.cu $(CSRC)/exact_scan.cu $(CSRC)/match_loop.cu $(CSRC)/tensor_scan.cu \
           $(CSRC)/flashmatch.cu $(CSRC)/comm.cu
CU_OBJ  := $(patsubst $(CSRC)/%.cu,build/cu/%.o,$(CU_SRC))
CU_HDR  := $(wildcard $(CSRC)/*.h $(CSRC)/*.cuh) include/fastnn_b200.h
HOST_SRC:= $(wildcard $(CSRC)/host/*.cpp)
HOST_OBJ:= $(patsubst $(CSRC)/host/%.cpp,build/host/%.o,$(HOST_SRC))
HOST_HDR:= $(wildcard include/fastnn/*.hpp $(CSRC)/host/*.hpp) include/fastnn_b200.h

LIB_CU  := $(PKG)/libfastnn_b200.so
LIB_CXX := $(PKG)/libfastnn.so
PYMOD   := $(PKG)/_fastnn$(EXT)

.PHONY: all product oracle testbins clean
all: product oracle testbins
product: $(LIB_CU) $(LIB_CXX) $(PYMOD)

# C++ test programs driving the drop-in library (run by tests/, -m gpu)
testbins: tests/cpp/c5_sharded
tests/cpp/c5_sharded: tests/cpp/c5_sharded.cpp $(LIB_CXX) $(HOST_HDR)
	g++ $(CXXFLAGS) -o $@ $< -L$(PKG) -lfastnn -lfastnn_b200 -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

build/cu/%.o: $(CSRC)/%.cu $(CU_HDR)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB_CU): $(CU_OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -Xlinker -soname=libfastnn_b200.so -ldl

build/host/%.o: $(CSRC)/host/%.cpp $(HOST_HDR)
	@mkdir -p $(dir $@)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIB_CXX): $(HOST_OBJ) $(LIB_CU)
	g++ -shared -o $@ $(HOST_OBJ) -L$(PKG) -lfastnn_b200 -Wl,-rpath,'$$ORIGIN' -Wl,-soname,libfastnn.so

$(PYMOD): $(CSRC)/bindings/module.cpp $(LIB_CXX) $(HOST_HDR)
	g++ $(CXXFLAGS) -I$(PYINC) -I$(PYBIND) -shared -o $@ $(CSRC)/bindings/module.cpp \
	    -L$(PKG) -lfastnn -lfastnn_b200 -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle PY=$(PY)

clean:
	rm -rf build $(LIB_CU) $(LIB_CXX) $(PYMOD)
