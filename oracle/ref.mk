# Builds the UNMODIFIED reference sources where they lie (/root/reference)
# against the committed Eigen / doctest shims: TEST INFRASTRUCTURE ONLY.
# Flags are the reference's Release build (proj/CMakeLists.txt:6-8: -O3,
# NDEBUG, no -march). Outputs go to oracle/_ref/ only (git-ignored, travels
# to the GPU box with the snapshot). Invoked by oracle/ref_build.sh.
REF ?= /root/reference/proj
OUT ?= _ref
JSON ?=
PRODUCT ?= ../paper_2511_03109_b200
CXX ?= g++
CXXFLAGS := -O3 -DNDEBUG -std=c++20 -fPIC -pthread -I$(REF)/include -I$(REF)/src -Ieigen_shim $(if $(JSON),-I$(JSON))
SRCS := common kernels geometry chebyshev tt farfield nearfield phmatrix serialize baselines harness
TESTS := kernels geometry chebyshev tt farfield nearfield phmatrix baselines
OBJS := $(SRCS:%=$(OUT)/obj/%.o) $(OUT)/obj/ref_driver.o

all: $(OUT)/libphmat_ref.so $(TESTS:%=$(OUT)/tests/test_%) $(if $(wildcard $(PRODUCT)/libphmat_b200.so),$(OUT)/dropin_check)

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

# Drop-in check: the reference's API and the product's C++ facade in one
# program (tests/cpp/dropin_check.cpp); needs the product library built.
$(OUT)/dropin_check: ../tests/cpp/dropin_check.cpp $(OUT)/libphmat_ref.so ../include/phmat_b200.hpp eigen_shim/Eigen/Dense
	$(CXX) $(CXXFLAGS) -I../include $< -o $@ -L$(OUT) -lphmat_ref -L$(PRODUCT) -lphmat_b200 \
	  -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,'$$ORIGIN/../../paper_2511_03109_b200'
