# Build recipe for the B200 matching engine and its CPU checkers.
#
#   make            -> paper_1303_1379_b200/libbmatch_b200.so  (sm_100a CUDA + host C-ABI)
#                      oracle/liboracle.so                      (C restatement of the reference path)
#   make ref        -> oracle/_ref/libbmatch_ref.so              (the reference compiled from its own
#                      sources under /root/reference; only where that tree exists)
#
# Built artefacts are git-ignored but travel to the GPU box with the gpurun snapshot.

NVCC      ?= nvcc
CXX       ?= g++
CC        ?= gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Xptxas -v \
             -Iinclude -Ipaper_1303_1379_b200/csrc
CXXFLAGS  := -O3 -std=c++17 -fPIC -Wall -Wextra -pthread -Iinclude
CFLAGS    := -O2 -std=c11 -fPIC -Wall -Wextra

PKG       := paper_1303_1379_b200
CSRC      := $(PKG)/csrc
BUILD     := build
LIB       := $(PKG)/libbmatch_b200.so
ORACLE    := oracle/liboracle.so
GENORACLE := oracle/libgen_oracle.so

REF_ROOT  ?= /root/reference/proj
REF_SRCS  := algorithms baselines csr_graph gpu_match kernel_grid matching matrix_market
# bench.cpp (run_suite) needs nlohmann/json, which the reference vendors but does not ship;
# the image has a copy inside cudnn_frontend. Without it the suite runner is left out.
NLOHMANN  ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann))
ifneq ($(NLOHMANN),)
REF_SRCS  += bench
REF_INC   := -I$(NLOHMANN)
endif
REF_LIB   := oracle/_ref/libbmatch_ref.so
SHIM_TEST := oracle/_ref/shim_test
SUITE     := oracle/_ref/b200_suite
SHIM_E2E  := oracle/_ref/shim_e2e

.PHONY: all ref shimtest suite clean
all: $(LIB) $(ORACLE) $(GENORACLE)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/bm_engine.o: $(CSRC)/bm_engine.cu $(CSRC)/bm_kernels.cuh $(CSRC)/bm_device.cuh include/bmatch_b200.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas.log || (cat $(BUILD)/ptxas.log; false)

$(BUILD)/bm_mg.o: $(CSRC)/bm_mg.cu $(CSRC)/bm_kernels.cuh $(CSRC)/bm_device.cuh include/bmatch_b200.h | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/ptxas_mg.log || (cat $(BUILD)/ptxas_mg.log; false)

$(BUILD)/bm_host.o: $(CSRC)/bm_host.cpp $(CSRC)/bm_host_util.hpp include/bmatch_b200.h include/bmatch_b200_gen.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/bm_io.o: $(CSRC)/bm_io.cpp $(CSRC)/bm_host_util.hpp include/bmatch_b200.h include/bmatch_b200_io.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(BUILD)/bm_engine.o $(BUILD)/bm_mg.o $(BUILD)/bm_host.o $(BUILD)/bm_io.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -pthread

$(ORACLE): oracle/bm_oracle.c oracle/bm_oracle.h
	$(CC) $(CFLAGS) -shared -o $@ oracle/bm_oracle.c

# the synthetic configs restated for the reference arm (no product library mapped)
$(GENORACLE): oracle/gen_oracle.cpp
	$(CXX) $(CXXFLAGS) -shared -o $@ $<

ref: $(REF_LIB)

$(REF_LIB): oracle/ref_capi.cpp $(foreach s,$(REF_SRCS),$(REF_ROOT)/src/$(s).cpp)
	mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O3 -DNDEBUG -fPIC -shared -pthread -I$(REF_ROOT)/include $(REF_INC) \
	    -o $@ oracle/ref_capi.cpp $(foreach s,$(REF_SRCS),$(REF_ROOT)/src/$(s).cpp)

# The C++ drop-in test: the reference's registry/driver/suite API calling the
# engine through include/bmatch_b200.hpp (needs the reference headers to build).
shimtest: $(SHIM_TEST)

$(SHIM_TEST): tests/cpp/shim_test.cpp include/bmatch_b200.hpp include/bmatch_b200.h $(REF_LIB) $(LIB)
	$(CXX) -std=c++20 -O2 -Wall -Wextra -pthread -I$(REF_ROOT)/include $(REF_INC) -Iinclude \
	    -o $@ tests/cpp/shim_test.cpp $(REF_LIB) $(LIB) \
	    -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,'$$ORIGIN/../../paper_1303_1379_b200'

# The paper's evaluation artefacts through the reference's run_suite (tools/b200_suite.cpp).
suite: $(SUITE) $(SHIM_E2E)

# The drop-in path's end-to-end time (reference types in, std::vector storage).
$(SHIM_E2E): tools/shim_e2e.cpp include/bmatch_b200.hpp include/bmatch_b200.h include/bmatch_b200_gen.h $(REF_LIB) $(LIB)
	$(CXX) -std=c++20 -O2 -Wall -Wextra -pthread -I$(REF_ROOT)/include $(REF_INC) -Iinclude \
	    -o $@ tools/shim_e2e.cpp $(REF_LIB) $(LIB) \
	    -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,'$$ORIGIN/../../paper_1303_1379_b200'

$(SUITE): tools/b200_suite.cpp include/bmatch_b200.hpp include/bmatch_b200.h include/bmatch_b200_gen.h $(REF_LIB) $(LIB)
	$(CXX) -std=c++20 -O2 -Wall -Wextra -pthread -I$(REF_ROOT)/include $(REF_INC) -Iinclude \
	    -o $@ tools/b200_suite.cpp $(REF_LIB) $(LIB) \
	    -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,'$$ORIGIN/../../paper_1303_1379_b200'

clean:
	rm -rf $(BUILD) $(LIB) $(ORACLE) $(GENORACLE)
