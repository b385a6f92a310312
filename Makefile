# Build the sm_100a engine (libqzcuda.so) and the test oracles.
#   make            engine + oracle
#   make ref        also compile the reference into oracle/_ref (needs /root/reference)
CUDA ?= /usr/local/cuda
NVCC ?= $(CUDA)/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -Xcompiler -Wall \
           -Xptxas -v
PKG := paper_2309_16979_b200
SRC := $(PKG)/csrc
OBJ := build/obj
LIB := $(PKG)/lib/libqzcuda.so
CU_SRCS := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
HDRS := $(wildcard $(SRC)/*.cuh) include/qzcuda.h
OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CPP_SRCS))

HOSTLIB := $(PKG)/lib/libqzsim_b200.so
TOOLS := build/tools/bench_transfer
HOST_SRCS := $(wildcard $(PKG)/host/*.cpp)
HOST_OBJS := $(patsubst $(PKG)/host/%.cpp,$(OBJ)/host_%.o,$(HOST_SRCS))
QZSIM_HDRS := $(wildcard include/qzsim/*.hpp) $(wildcard $(PKG)/host/*.hpp)

all: $(LIB) $(HOSTLIB) oracle $(TOOLS)

$(OBJ)/host_%.o: $(PKG)/host/%.cpp $(QZSIM_HDRS) include/qzcuda.h
	@mkdir -p $(OBJ)
	g++ -std=gnu++20 -O2 -fPIC -Wall -Iinclude -c $< -o $@

# The C++ drop-in layer (include/qzsim/*.hpp) over the C ABI.
$(HOSTLIB): $(HOST_OBJS) $(LIB)
	g++ -shared -o $@ $(HOST_OBJS) -L$(PKG)/lib -lqzcuda -Wl,-rpath,'$$ORIGIN'


$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

# the device headers the runtime-specialised passes compile against (NVRTC),
# embedded as raw strings
JIT_HDRS := $(SRC)/qz_rtc_types.cuh $(SRC)/qz_bits.cuh $(SRC)/qz_gate_types.cuh $(SRC)/qz_gates_dev.cuh
$(OBJ)/jit_headers.inc: $(JIT_HDRS)
	@mkdir -p $(OBJ)
	@{ echo "static const int kJitHeaderCount = 4;"; \
	   echo "static const char *const kJitHeaderNames[] = {"; \
	   for f in $(JIT_HDRS); do echo "\"$$(basename $$f)\","; done; echo "};"; \
	   echo "static const char *const kJitHeaderSrc[] = {"; \
	   for f in $(JIT_HDRS); do echo 'R"QZSRC('; cat $$f; echo ')QZSRC",'; done; echo "};"; } > $@

$(OBJ)/qz_jit.o: $(SRC)/qz_jit.cu $(HDRS) $(OBJ)/jit_headers.inc
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -I$(OBJ) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	g++ -std=c++17 -O2 -fPIC -Wall -I$(CUDA)/include -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart -ldl

# tools over the drop-in (paper Table 1: tools/cpp/bench_transfer.cpp)
build/tools/bench_transfer: tools/cpp/bench_transfer.cpp $(HOSTLIB) $(QZSIM_HDRS)
	@mkdir -p build/tools
	g++ -std=gnu++20 -O2 -Iinclude $< -o $@ -L$(PKG)/lib -lqzsim_b200 -lqzcuda -Wl,-rpath,'$$ORIGIN/../../$(PKG)/lib'

tools: $(TOOLS)

oracle:
	$(MAKE) -C oracle all

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(PKG)/lib oracle/liboracle.so

.PHONY: all oracle ref clean tools
