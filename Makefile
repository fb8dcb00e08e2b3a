# Top-level build: the product library (host C++ + sm_100a CUDA), the
# oracle checkers, and the reference-test drivers.  __graft_entry__.build()
# runs `make -j`.  Outputs (git-ignored, shipped to the GPU box with gpurun):
#   paper_2510_02676_b200/lib/libecf8_b200.so   product: C ABI + C++ API
#   oracle/_build/liboracle.so, oracle/_ref/...  checkers (oracle/Makefile)
#   build/ref_unit_tests, build/ref_acceptance   reference suites linked
#                                                against the product library

CUDA    ?= /usr/local/cuda
NVCC    := $(CUDA)/bin/nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
PKG     := paper_2510_02676_b200
LIBDIR  := $(PKG)/lib
OBJ     := build/obj
LIB     := $(LIBDIR)/libecf8_b200.so

CXXFLAGS  := -std=c++20 -O3 -fPIC -fopenmp -Wall -Wextra -Iinclude -I$(CUDA)/include
NVCCFLAGS := -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC,-fopenmp -Xptxas -v \
             -Iinclude -I$(PKG)/csrc/cuda --expt-relaxed-constexpr $(EXTRA)

HOST_SRCS := $(wildcard $(PKG)/csrc/host/*.cpp) $(PKG)/csrc/cuda/tables.cpp
CU_SRCS   := $(wildcard $(PKG)/csrc/cuda/*.cu)
HOST_OBJS := $(patsubst $(PKG)/csrc/%.cpp,$(OBJ)/%.o,$(HOST_SRCS))
CU_OBJS   := $(patsubst $(PKG)/csrc/%.cu,$(OBJ)/%.o,$(CU_SRCS))
HEADERS   := $(wildcard include/*.h include/ecf8/*.hpp $(PKG)/csrc/host/*.hpp $(PKG)/csrc/cuda/*.hpp $(PKG)/csrc/cuda/*.cuh)

all: $(LIB) oracle refsuites

$(OBJ)/%.o: $(PKG)/csrc/%.cpp $(HEADERS)
	@mkdir -p $(dir $@)
	g++ $(CXXFLAGS) -c $< -o $@

$(OBJ)/%.o: $(PKG)/csrc/%.cu $(HEADERS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVCCFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(HOST_OBJS) $(CU_OBJS)
	@mkdir -p $(dir $@)
	g++ -shared -o $@ $^ -fopenmp -L$(CUDA)/lib64 -lcudart_static -ldl -lrt -lpthread \
	    -Wl,--no-undefined

oracle:
	$(MAKE) -C oracle

# A/B kernel experiments: make variant V=name VFLAGS="-DECF8_WB_DEPTH=4"
# -> build/var/name/libecf8_b200.so (load with ECF8_LIB=...)
variant:
	$(MAKE) OBJ=build/var/$(V)/obj LIB=build/var/$(V)/libecf8_b200.so EXTRA="$(VFLAGS)" build/var/$(V)/libecf8_b200.so

# The reference's own unit + acceptance suites, compiled from
# /root/reference/proj/tests (never copied) against OUR headers and library.
REF_TESTS := /root/reference/proj/tests
JSON_INC  ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
ifneq ($(wildcard $(REF_TESTS)/test_codec.cpp),)
refsuites: build/ref_unit_tests build/ref_acceptance
build/ref_unit_tests: $(LIB) tests/cpp/doctest.h $(wildcard $(REF_TESTS)/*.cpp)
	@mkdir -p build
	g++ -std=c++20 -O2 -Iinclude -Itests/cpp -I$(REF_TESTS) -I$(JSON_INC) -o $@ \
	    $(REF_TESTS)/test_main.cpp $(REF_TESTS)/test_fp8.cpp $(REF_TESTS)/test_entropy.cpp \
	    $(REF_TESTS)/test_huffman.cpp $(REF_TESTS)/test_lut.cpp $(REF_TESTS)/test_codec.cpp \
	    $(REF_TESTS)/test_container.cpp -L$(LIBDIR) -lecf8_b200 -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)'
build/ref_acceptance: $(LIB) $(REF_TESTS)/acceptance.cpp
	@mkdir -p build
	g++ -std=c++20 -O2 -Iinclude -I$(REF_TESTS) -o $@ $(REF_TESTS)/acceptance.cpp \
	    -L$(LIBDIR) -lecf8_b200 -Wl,-rpath,'$$ORIGIN/../$(LIBDIR)'
else
refsuites:
	@echo "reference tests absent: build/ref_* not rebuilt"
endif

clean:
	rm -rf build $(LIBDIR)
	$(MAKE) -C oracle clean

.PHONY: all oracle refsuites clean variant
