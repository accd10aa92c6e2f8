# c3-b200 build: everything in-tree so the built .so files travel to the GPU box.
#
#   paper_2412_14335_b200/lib/libc3sim.so   C++ model layer behind include/c3sim/*.hpp
#   paper_2412_14335_b200/lib/libc3cuda.so  sm_100a CUDA kernels + C3 runtime behind
#                                           the C-ABI include/c3cuda.h (and the C++
#                                           execution API include/c3sim/exec.hpp)
#   paper_2412_14335_b200/bin/c3sim         product CLI (reference tools/c3sim_main.cpp surface)
#   oracle/                                 test-only oracle (make -C oracle)

CXX      := g++-13
NVCC     ?= /usr/local/cuda/bin/nvcc
CUDA     ?= /usr/local/cuda
JSON_DIR ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
PKG      := paper_2412_14335_b200
LIB      := $(PKG)/lib
BIN      := $(PKG)/bin
OBJ      := build/obj
ARCH     := -gencode arch=compute_100a,code=sm_100a

CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(JSON_DIR)
NVFLAGS  := -std=c++17 -O3 $(ARCH) $(NVCC_EXTRA) -lineinfo -Xcompiler -fPIC -Iinclude -I$(PKG)/csrc/cuda \
            --expt-relaxed-constexpr -ccbin $(CXX) -Xptxas -v

MODEL_SRC := $(wildcard $(PKG)/csrc/model/*.cpp)
MODEL_OBJ := $(patsubst $(PKG)/csrc/model/%.cpp,$(OBJ)/model/%.o,$(MODEL_SRC))
CU_SRC    := $(wildcard $(PKG)/csrc/cuda/*.cu)
CU_OBJ    := $(patsubst $(PKG)/csrc/cuda/%.cu,$(OBJ)/cuda/%.o,$(CU_SRC))
CC_SRC    := $(wildcard $(PKG)/csrc/cuda/*.cpp)
CC_OBJ    := $(patsubst $(PKG)/csrc/cuda/%.cpp,$(OBJ)/cuda/%.o,$(CC_SRC))
CU_HDR    := $(wildcard $(PKG)/csrc/cuda/*.cuh) $(wildcard $(PKG)/csrc/cuda/*.hpp) include/c3cuda.h

PYINC    := $(shell python3 -c "import sysconfig; print(sysconfig.get_paths()['include'])")
PYBIND   := $(shell python3 -c "import pybind11; print(pybind11.get_include())")
PYEXT    := $(shell python3 -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
PYMOD    := $(PKG)/python/c3sim/_c3sim$(PYEXT)

.PHONY: all model cuda cli python oracle clean
all: model cuda cli python oracle
model: $(LIB)/libc3sim.so
cuda: $(LIB)/libc3cuda.so
cli: $(BIN)/c3sim
python: $(PYMOD)
oracle:
	$(MAKE) -C oracle -s

$(OBJ)/model/%.o: $(PKG)/csrc/model/%.cpp $(wildcard include/c3sim/*.hpp)
	@mkdir -p $(@D)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB)/libc3sim.so: $(MODEL_OBJ)
	@mkdir -p $(@D)
	$(CXX) -shared -o $@ $^

$(OBJ)/cuda/%.o: $(PKG)/csrc/cuda/%.cu $(CU_HDR)
	@mkdir -p $(@D)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/cuda/$*.ptxas.txt || (cat $(OBJ)/cuda/$*.ptxas.txt; false)

$(OBJ)/cuda/%.o: $(PKG)/csrc/cuda/%.cpp $(CU_HDR) $(wildcard include/c3sim/*.hpp)
	@mkdir -p $(@D)
	$(CXX) $(CXXFLAGS) -I$(CUDA)/include -I$(PKG)/csrc/cuda -c $< -o $@

$(LIB)/libc3cuda.so: $(CU_OBJ) $(CC_OBJ) $(LIB)/libc3sim.so
	@mkdir -p $(@D)
	$(NVCC) $(ARCH) -shared -ccbin $(CXX) -o $@ $(CU_OBJ) $(CC_OBJ) -L$(LIB) -lc3sim \
	    -lcudart_static -Xlinker -rpath,'$$ORIGIN'

$(BIN)/c3sim: $(PKG)/csrc/tools/c3sim_cli.cpp $(LIB)/libc3sim.so $(LIB)/libc3cuda.so include/c3sim/exec.hpp
	@mkdir -p $(@D)
	$(CXX) $(CXXFLAGS) $< -L$(LIB) -lc3cuda -lc3sim -Wl,-rpath,'$$ORIGIN/../lib' -o $@

# pybind11 module: the reference's Python surface over the product libraries
$(PYMOD): $(PKG)/csrc/python/c3sim_module.cpp $(LIB)/libc3sim.so $(LIB)/libc3cuda.so $(wildcard include/c3sim/*.hpp)
	@mkdir -p $(@D)
	$(CXX) $(CXXFLAGS) -Wno-unused-parameter -shared -I$(PYINC) -I$(PYBIND) $< -L$(LIB) -lc3cuda -lc3sim \
	    -Wl,-rpath,'$$ORIGIN/../../lib' -o $@

clean:
	rm -rf build $(LIB) $(BIN)
