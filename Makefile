# Top-level build: the sm_100a CUDA library behind include/dfs_gpu.h, the C++
# drop-in shim (include/dfs/*.hpp), and the test-only oracle.
#
#   make            -> paper_2605_23445_b200/libdfs_b200.so (+ oracle)
#   make oracle-ref -> oracle/_ref/libdfsref.so (needs /root/reference)

NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2605_23445_b200
CSRC     := $(PKG)/csrc
OBJDIR   := build/obj
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -I$(CSRC) \
            --expt-relaxed-constexpr -Xptxas -v
CU_SRCS  := $(wildcard $(CSRC)/*.cu)
CU_OBJS  := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
SHIM_SRCS:= $(wildcard $(CSRC)/*.cpp)
SHIM_OBJS:= $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.cpp.o,$(SHIM_SRCS))

.PHONY: all lib oracle oracle-ref clean
all: lib oracle

lib: $(PKG)/libdfs_b200.so

$(OBJDIR)/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh include/dfs_gpu.h $(wildcard $(CSRC)/*.cuh)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.log || (cat $@.log; false)

$(OBJDIR)/%.cpp.o: $(CSRC)/%.cpp include/dfs_gpu.h $(wildcard include/dfs/*.hpp)
	@mkdir -p $(OBJDIR)
	g++ -std=c++20 -O2 -fPIC -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(PKG)/libdfs_b200.so: $(CU_OBJS) $(SHIM_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart -lcuda

oracle:
	$(MAKE) -s -C oracle

oracle-ref:
	$(MAKE) -s -C oracle ref

clean:
	rm -rf build $(PKG)/libdfs_b200.so
