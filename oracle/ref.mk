# Builds the UNMODIFIED reference sources where they lie (/root/reference)
# against the committed Eigen / doctest shims: TEST INFRASTRUCTURE ONLY.
# Flags are the reference's Release build (proj/CMakeLists.txt:6-8: -O3,
# NDEBUG, no -march). Outputs go to oracle/_ref/ only (git-ignored, travels
# to the GPU box with the snapshot). Invoked by oracle/ref_build.sh.
REF ?= /root/reference/proj
OUT ?= _ref
JSON ?=
CXX ?= g++
CXXFLAGS := -O3 -DNDEBUG -std=c++20 -fPIC -pthread -I$(REF)/include -I$(REF)/src -Ieigen_shim $(if $(JSON),-I$(JSON))
SRCS := common kernels geometry chebyshev tt farfield nearfield phmatrix serialize baselines harness
TESTS := kernels geometry chebyshev tt farfield nearfield phmatrix baselines
OBJS := $(SRCS:%=$(OUT)/obj/%.o) $(OUT)/obj/ref_driver.o

all: $(OUT)/libphmat_ref.so $(TESTS:%=$(OUT)/tests/test_%)

$(OUT)/obj/%.o: $(REF)/src/%.cpp eigen_shim/Eigen/Dense
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/obj/ref_driver.o: ref_driver.cpp eigen_shim/Eigen/Dense
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/libphmat_ref.so: $(OBJS)
	$(CXX) -shared -pthread -o $@ $(OBJS)

$(OUT)/tests/test_%: $(REF)/tests/test_%.cpp $(OUT)/libphmat_ref.so doctest_shim/doctest.h
	@mkdir -p $(OUT)/tests
	$(CXX) $(CXXFLAGS) -Idoctest_shim $< -o $@ -L$(OUT) -lphmat_ref -Wl,-rpath,'$$ORIGIN/..'

.PHONY: all
