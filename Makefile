# Build the sm_100a engine library in-tree (travels to the GPU box with the repo).
# Translation units compile in parallel (make -j); the library links them.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude
LIB := paper_2210_15874_b200/lib/libqtn_b200.so
CSRC := paper_2210_15874_b200/csrc
SRC := $(CSRC)/qtn_b200.cu $(CSRC)/bucket_strided.cu $(CSRC)/bucket_expand.cu $(CSRC)/bucket_stream.cu $(CSRC)/planner.cpp $(CSRC)/plan_template.cpp
# K6 (bucket_fused.cu): one source, three objects — planner + C ABI, complex64
# kernels, complex128 kernels — so the kernel halves compile in parallel
K6PARTS := 0 1 2
OBJDIR := build/obj
HDRS := include/qtn_b200.h $(CSRC)/knobs.h $(CSRC)/k4_plan.h
OBJ := $(patsubst $(CSRC)/%,$(OBJDIR)/%.o,$(SRC)) $(foreach i,$(K6PARTS),$(OBJDIR)/bucket_fused_$(i).o)
DBGOBJ := $(patsubst $(CSRC)/%,$(OBJDIR)/debug/%.o,$(SRC)) $(foreach i,$(K6PARTS),$(OBJDIR)/debug/bucket_fused_$(i).o)

all: $(LIB)

$(OBJDIR)/%.o: $(CSRC)/% $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) $(EXTRA) -c -o $@ $<

$(OBJDIR)/bucket_fused_%.o: $(CSRC)/bucket_fused.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) $(EXTRA) -DK6_PART=$* -c -o $@ $<

$(OBJDIR)/debug/%.o: $(CSRC)/% $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DQTN_DEBUG -c -o $@ $<

$(OBJDIR)/debug/bucket_fused_%.o: $(CSRC)/bucket_fused.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -DQTN_DEBUG -DK6_PART=$* -c -o $@ $<

$(LIB): $(OBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

# variant build for A/B measurements: make variant TAG=x EXTRA="-DFOO" -> lib/libqtn_b200_x.so
variant:
	$(MAKE) OBJDIR=build/obj_$(TAG) EXTRA="$(EXTRA)" LIB=paper_2210_15874_b200/lib/libqtn_b200_$(TAG).so

# bounds-checked build (device asserts), for GPU debugging without compute-sanitizer
debug: $(DBGOBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o paper_2210_15874_b200/lib/libqtn_b200_debug.so $(DBGOBJ)

sass: $(LIB)
	cuobjdump -sass $(LIB) | grep -E "Function|LDG|STG|ATOM|RED" | head -50

clean:
	rm -rf $(LIB) build

.PHONY: all clean sass variant debug
