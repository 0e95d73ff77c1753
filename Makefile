# Builds the product library (sm_100a) and the CPU checkers.
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG       := paper_1609_07228_b200
SRCS      := $(wildcard $(PKG)/csrc/*.cu)
OBJS      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
LIB       := $(PKG)/libannkit_b200.so

FACADE    := $(PKG)/libannkit_facade.so
FACADE_T  := tests/cpp/test_facade
FACADE_SRCS := $(PKG)/cpp/annkit_facade.cpp $(PKG)/cpp/annkit_io.cpp

all: $(LIB) $(FACADE) $(FACADE_T) oracle refsuite

build/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh) include/annkit_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS)

# C++ host API (include/annkit_b200.hpp) over the C-ABI, and its test program
$(FACADE): $(FACADE_SRCS) include/annkit_b200.hpp include/annkit_b200.h $(LIB)
	g++ -std=c++20 -O2 -fPIC -shared -Wall -Iinclude -o $@ $(FACADE_SRCS) -L$(PKG) -lannkit_b200 -Wl,-rpath,'$$ORIGIN'

$(FACADE_T): tests/cpp/test_facade.cpp include/annkit_b200.hpp $(FACADE)
	g++ -std=c++20 -O2 -Wall -Iinclude -o $@ $< -L$(PKG) -lannkit_facade -lannkit_b200 \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

oracle:
	$(MAKE) -C oracle

# The reference's own unit suites and acceptance runner, compiled UNCHANGED from
# /root/reference/proj/tests against include/annkit_b200.hpp (tests/cpp/shim maps
# <doctest.h> and "annkit/*.hpp" to our headers) and linked to the facade.  Built
# only where /root/reference exists; the binaries travel to the GPU box.
REFT      ?= /root/reference/proj/tests
REFSUITE  := tests/cpp/_refsuite
refsuite:
	@if [ -d "$(REFT)" ]; then $(MAKE) $(REFSUITE)/unit $(REFSUITE)/acceptance; \
	else echo "reference tests absent; keeping prebuilt $(REFSUITE)/ (if any)"; fi

REFT_UNIT := $(addprefix $(REFT)/,doctest_main.cpp test_dataset.cpp test_eval.cpp test_graph_build.cpp test_kd_forest.cpp test_search.cpp)
$(REFSUITE)/unit: $(REFT_UNIT) tests/cpp/doctest/doctest.h include/annkit_b200.hpp $(FACADE)
	@mkdir -p $(REFSUITE)
	g++ -std=c++20 -O2 -w -Itests/cpp/doctest -Itests/cpp/shim -Iinclude -I$(REFT) -o $@ $(REFT_UNIT) -L$(PKG) -lannkit_facade \
	    -lannkit_b200 -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'
$(REFSUITE)/acceptance: $(REFT)/acceptance.cpp include/annkit_b200.hpp $(FACADE)
	@mkdir -p $(REFSUITE)
	g++ -std=c++20 -O2 -w -Itests/cpp/doctest -Itests/cpp/shim -Iinclude -I$(REFT) -o $@ $(REFT)/acceptance.cpp -L$(PKG) \
	    -lannkit_facade -lannkit_b200 -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'

clean:
	rm -rf build $(LIB) $(FACADE) $(FACADE_T)
	$(MAKE) -C oracle clean

.PHONY: all oracle refsuite clean

# device-debug build for compute-sanitizer sessions (not used by tests/bench)
debug: $(SRCS)
	@mkdir -p build/dbg
	for f in $(SRCS); do $(NVCC) -O2 -lineinfo -DANNK_DEBUG_CHECKS -std=c++17 $(ARCH) -Xcompiler -fPIC --expt-relaxed-constexpr -c $$f -o build/dbg/$$(basename $$f .cu).o || exit 1; done
	$(NVCC) $(ARCH) -shared -cudart static -o build/libannkit_b200_dbg.so build/dbg/*.o
