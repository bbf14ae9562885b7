# Build the sm_100a engine library in-tree (travels to the GPU box with the repo).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static -Iinclude
LIB := paper_2210_15874_b200/lib/libqtn_b200.so
SRC := paper_2210_15874_b200/csrc/qtn_b200.cu paper_2210_15874_b200/csrc/bucket_strided.cu paper_2210_15874_b200/csrc/planner.cpp paper_2210_15874_b200/csrc/plan_template.cpp

all: $(LIB)

$(LIB): $(SRC) include/qtn_b200.h
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -o $@ $(SRC)

# variant build for A/B measurements: make variant TAG=x EXTRA="-DFOO" -> lib/libqtn_b200_x.so
variant:
	$(NVCC) $(NVFLAGS) $(EXTRA) -o paper_2210_15874_b200/lib/libqtn_b200_$(TAG).so $(SRC)

# bounds-checked build (device asserts), for GPU debugging without compute-sanitizer
debug:
	$(NVCC) $(NVFLAGS) -DQTN_DEBUG -o paper_2210_15874_b200/lib/libqtn_b200_debug.so $(SRC)

sass: $(LIB)
	cuobjdump -sass $(LIB) | grep -E "Function|LDG|STG|ATOM|RED" | head -50

clean:
	rm -f $(LIB)

.PHONY: all clean sass
