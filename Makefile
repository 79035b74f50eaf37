# Builds the product library paper_2311_01635_b200/librtpb.so (sm_100a only)
# and the CPU oracle (oracle/, test infrastructure).
NVCC    ?= /usr/local/cuda/bin/nvcc
SITE    ?= $(shell python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])" 2>/dev/null)
NCCL_DIR ?= $(SITE)/nvidia/nccl
PKG     := paper_2311_01635_b200
CSRC    := $(PKG)/csrc
OBJDIR  ?= build/obj
OUT     ?= $(PKG)/librtpb.so
# EXTRA: extra nvcc/g++ defines for A/B builds (tools/build_variant.sh)
EXTRA   ?=
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr \
           -Iinclude -I$(CSRC) -I$(NCCL_DIR)/include -Xptxas -v $(EXTRA)
CXX     ?= g++
CXXFLAGS := -std=c++20 -O2 -g -fPIC -Wall -Wextra -Wno-unused-parameter -Iinclude -I$(CSRC) \
            -I/usr/local/cuda/include -I$(NCCL_DIR)/include $(EXTRA)
CU_SRC  := $(CSRC)/kernels/gemm_launch.cu $(CSRC)/kernels/elementwise.cu $(CSRC)/kernels/attention.cu \
           $(CSRC)/kernels/moe_embed.cu \
           $(CSRC)/capi_steps.cu
CPP_SRC := $(wildcard $(CSRC)/host/*.cpp)
OBJS    := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRC)) $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.o,$(CPP_SRC))
HDRS    := $(wildcard include/*.h include/rtpb/*.hpp $(CSRC)/kernels/*.cuh $(CSRC)/kernels/*.hpp $(CSRC)/host/*.hpp)

.PHONY: all lib oracle cpptest clean
all: lib oracle cpptest
lib: $(OUT)
oracle:
	$(MAKE) -s -C oracle oracle

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.log || (cat $@.log; false)

$(OBJDIR)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT): $(OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath,$(NCCL_DIR)/lib -lpthread

# The C++ drop-in test: a reference-style caller compiled against include/rtpb/rtp.hpp only.
cpptest: build/dropin_test
build/dropin_test: tests/cpp/dropin_test.cpp include/rtpb/rtp.hpp include/rtpb.h $(OUT)
	@mkdir -p build
	$(CXX) -std=c++20 -O1 -g -Wall -Wextra -Iinclude $< -o $@ -L$(PKG) -lrtpb -Wl,-rpath,'$$ORIGIN/../$(PKG)'

clean:
	rm -rf build $(PKG)/librtpb.so
