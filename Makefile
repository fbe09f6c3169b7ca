# Builds the product library paper_2505_00982_b200/libdho2gpu.so (sm_100a only) and the
# test-only CPU checkers under oracle/ (see oracle/Makefile).
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -O3 --expt-relaxed-constexpr
PKG      := paper_2505_00982_b200
SRCS     := $(wildcard $(PKG)/csrc/*.cu)
OBJS     := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
HDRS     := $(wildcard $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh) include/dho2gpu.h
LIB      := $(PKG)/libdho2gpu.so

all: $(LIB) oracle dropin

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static -ldl -lpthread -lrt

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

oracle:
	$(MAKE) -C oracle oracle
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C oracle ref; fi

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

# the reference-side drop-in test binary (needs the reference objects and the library)
dropin: $(LIB) oracle
	@if [ -d /root/reference/proj/src ]; then $(MAKE) -C integration; fi

.PHONY: all oracle dropin clean
