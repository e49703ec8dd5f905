# Build libwm3.so (sm_100a only) and the oracle's C helpers.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -v $(NVFLAGS_EXTRA)
PKG := paper_2503_22235_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/wm3.h
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))

all: $(PKG)/libwm3.so

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libwm3.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

# profiling aid outside the public ABI (tools/mma_probe.py)
probe: tools/libmma_probe.so
tools/libmma_probe.so: tools/csrc/mma_probe.cu $(PKG)/libwm3.so
	$(NVCC) $(NVFLAGS) -shared -o $@ $< $(PKG)/libwm3.so -lcuda

clean:
	rm -rf build $(PKG)/libwm3.so tools/libmma_probe.so

.PHONY: all clean probe
