# B200 build of the Hydra shard-execution path.
#   make            -> paper_2110_08633_b200/libhydra.so (host C++ + sm_100a kernels + C-ABI)
#                      build/plan_dump_b200 (parity driver compiled against this build)
#                      oracle/liboracle_gpt.so (CPU numeric oracle — test infrastructure)
#   make ref        -> oracle/_ref/* (reference compiled from /root/reference; needs the tree)
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      := /usr/bin/g++
NLOHMANN ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
CUDA_INC := /usr/local/cuda/include
PKG      := paper_2110_08633_b200
CSRC     := $(PKG)/csrc
B        := build

CXXFLAGS  := -std=c++20 -O2 -fPIC -g -Wall -Wextra -Wno-dangling-reference -Wno-unused-parameter -Iinclude -I$(NLOHMANN) -I$(CUDA_INC) -pthread -fopenmp
NVFLAGS   := -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a \
             -Iinclude -I$(CSRC)/kernels --expt-relaxed-constexpr -Xptxas -v

HOST_SRCS := $(wildcard $(CSRC)/host/*.cpp)
EXEC_SRCS := $(wildcard $(CSRC)/exec/*.cpp)
CAPI_SRCS := $(wildcard $(CSRC)/capi/*.cpp)
CU_SRCS   := $(wildcard $(CSRC)/kernels/*.cu)
HOST_OBJS := $(patsubst $(CSRC)/%.cpp,$(B)/%.o,$(HOST_SRCS) $(EXEC_SRCS) $(CAPI_SRCS))
CU_OBJS   := $(patsubst $(CSRC)/%.cu,$(B)/%.o,$(CU_SRCS))
HDRS      := $(wildcard include/*.h include/spillsim/*.hpp $(CSRC)/kernels/*.cuh $(CSRC)/exec/*.hpp)

all: $(PKG)/libhydra.so $(B)/plan_dump_b200 $(B)/test_spillsim oracle/liboracle_gpt.so

$(B)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

# host optimizer: vectorised AdamW (sqrt without errno so it vectorises)
$(B)/exec/host_opt.o: CXXFLAGS += -O3 -fno-math-errno

$(B)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(PKG)/libhydra.so: $(HOST_OBJS) $(CU_OBJS)
	$(CXX) -shared $^ -o $@ -Wl,-Bsymbolic -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -pthread \
	  -L/usr/lib/gcc/x86_64-linux-gnu/13 -lgomp

$(B)/plan_dump_b200: oracle/plan_dump.cpp $(PKG)/libhydra.so
	$(CXX) $(CXXFLAGS) $< -o $@ -L$(PKG) -lhydra -Wl,-rpath,'$$ORIGIN/../$(PKG)'

$(B)/test_spillsim: tests/native/test_spillsim.cpp $(PKG)/libhydra.so
	$(CXX) $(CXXFLAGS) $< -o $@ -L$(PKG) -lhydra -Wl,-rpath,'$$ORIGIN/../$(PKG)'

oracle/liboracle_gpt.so: oracle/gpt_oracle.c oracle/gpt_oracle.h
	gcc -std=gnu11 -O3 -fPIC -fopenmp -shared $< -o $@ -lm

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf $(B) $(PKG)/libhydra.so oracle/liboracle_gpt.so

.PHONY: all ref clean
