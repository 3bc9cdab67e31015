# Builds the C-ABI executor library in-tree (it travels to the GPU box with
# the snapshot).  sm_100a only.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
PKG := paper_1701_03980_b200
SRC := $(PKG)/csrc
OBJ := build/obj
LIB := $(PKG)/libdyngpu.so
OBJS := $(OBJ)/executor.o $(OBJ)/kernels.o $(OBJ)/gemm.o $(OBJ)/tcgemm.o $(OBJ)/rnn.o $(OBJ)/tmagemm.o $(OBJ)/cellgemm.o

PYTHON ?= python3
PYINC := $(shell $(PYTHON) -c "import sysconfig; print(sysconfig.get_paths()['include'])")
PYEXT := $(shell $(PYTHON) -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
CORE := $(PKG)/_dgcore$(PYEXT)

all: $(LIB) $(CORE)

# host-side native graph construction (CPython extension, plain C)
$(CORE): $(SRC)/dgcore.c
	gcc -O2 -Wall -shared -fPIC -I$(PYINC) $< -o $@

$(OBJ):
	mkdir -p $(OBJ)

$(OBJ)/executor.o: $(SRC)/executor.cpp $(SRC)/kernels.cuh include/dyngpu.h | $(OBJ)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(OBJ)/kernels.o: $(SRC)/kernels.cu $(SRC)/kernels.cuh | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/gemm.o: $(SRC)/gemm.cu $(SRC)/kernels.cuh | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/tcgemm.o: $(SRC)/tcgemm.cu $(SRC)/kernels.cuh | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/tmagemm.o: $(SRC)/tmagemm.cu $(SRC)/kernels.cuh | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/cellgemm.o: $(SRC)/cellgemm.cu $(SRC)/kernels.cuh | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/rnn.o: $(SRC)/rnn.cu $(SRC)/kernels.cuh | $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart_static -lrt -ldl -lpthread

clean:
	rm -rf build $(LIB) $(CORE)

.PHONY: all clean
