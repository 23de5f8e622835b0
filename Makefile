# B200-native siting engine: one shared library with the sm_100a kernels and
# the C-ABI (include/txsite_b200.h), the C++ host API + CLI on top of it, and
# the CPU oracle (test infrastructure, oracle/Makefile).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -Wall -Xptxas -warn-spills
PKG := paper_2006_16783_b200
BUILD := build
CU_SRC := $(wildcard $(PKG)/csrc/*.cu)
CPP_SRC := $(wildcard $(PKG)/csrc/*.cpp)
HDRS := $(wildcard $(PKG)/csrc/*.hpp $(PKG)/csrc/*.cuh) include/txsite_b200.h
OBJ := $(CU_SRC:$(PKG)/csrc/%.cu=$(BUILD)/%.o) $(CPP_SRC:$(PKG)/csrc/%.cpp=$(BUILD)/%.cpp.o)
LIB := $(PKG)/libtxsite_b200.so
CHECKED := $(PKG)/libtxsite_b200_checked.so
CHK_OBJ := $(CU_SRC:$(PKG)/csrc/%.cu=$(BUILD)/chk_%.o) $(CPP_SRC:$(PKG)/csrc/%.cpp=$(BUILD)/chk_%.cpp.o)

HOSTLIB := $(PKG)/libtxsite_host.so
CLI := $(PKG)/bin/txsite
APICHK := $(PKG)/bin/txsite_api_check

all: $(LIB) $(CHECKED) $(HOSTLIB) $(CLI) $(APICHK) oracle

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(PKG)/csrc/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/%.cpp.o: $(PKG)/csrc/%.cpp $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -ldl

# bounds-checked variant for the tests (terrain loads trap when out of range)
$(BUILD)/chk_%.o: $(PKG)/csrc/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -DTXS_BOUNDS_CHECK -c $< -o $@
$(BUILD)/chk_%.cpp.o: $(PKG)/csrc/%.cpp $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -DTXS_BOUNDS_CHECK -x cu -c $< -o $@
$(CHECKED): $(CHK_OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(CHK_OBJ) -ldl

$(HOSTLIB): $(PKG)/host/txsite.cpp include/txsite/txsite.hpp include/txsite_b200.h $(LIB)
	g++ -std=c++17 -O2 -fPIC -shared -Wall -Wextra -Iinclude -o $@ $(PKG)/host/txsite.cpp -L$(PKG) -ltxsite_b200 -Wl,-rpath,'$$ORIGIN'

$(CLI): $(PKG)/host/txsite_main.cpp $(HOSTLIB)
	mkdir -p $(PKG)/bin
	g++ -std=c++17 -O2 -Wall -Wextra -Iinclude -o $@ $(PKG)/host/txsite_main.cpp -L$(PKG) -ltxsite_host -ltxsite_b200 -Wl,-rpath,'$$ORIGIN/..'

# the reference-shaped C++ value-type API exercised end to end (tests/test_gpu_cli.py)
$(APICHK): tests/cpp/api_check.cpp $(HOSTLIB)
	mkdir -p $(PKG)/bin
	g++ -std=c++17 -O2 -Wall -Wextra -Iinclude -o $@ tests/cpp/api_check.cpp -L$(PKG) -ltxsite_host -ltxsite_b200 -Wl,-rpath,'$$ORIGIN/..'

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(LIB) $(CHECKED) $(HOSTLIB) $(CLI) $(APICHK)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
