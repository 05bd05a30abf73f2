# TEST INFRASTRUCTURE ONLY: builds the REFERENCE's own MIDBF code, unmodified
# from /root/reference/proj/src, against the Eigen / doctest stand-ins in
# oracle/shim/ (Eigen3 and the vendor/ doctest are absent from this image;
# gmpxx too, so the Delaunay recovery geometry, src/delaunay.cpp, is not
# built and its callers are left unresolved), into oracle/_ref/:
#   libmidbf_ref.so  reference sources + oracle/ref_capi.cpp (C ABI for tests)
#   ref_unit_tests   the reference's own doctest suites for the hot path
#                    (tests/test_{butterfly,linalg,tree,kernels}.cpp)
# Flags follow the reference's release build (proj/CMakeLists.txt:11: -O2,
# C++20, OpenMP).  Run from the repo root: make -f oracle/ref.mk
# Needs /root/reference (this container); the GPU box uses the built files.
REF ?= /root/reference/proj
CXX := /usr/bin/g++
OUT := oracle/_ref
CXXFLAGS := -O2 -std=c++20 -fPIC -fopenmp -Ioracle/shim -I$(REF)/include -w
SRC := tree linalg butterfly butterfly_io geometry kernels metrics phase_md phase1d
TESTS := main test_butterfly test_linalg test_tree test_kernels
SHIM := oracle/shim/midbf_eigen_shim.hpp oracle/shim/doctest.h
OBJ := $(patsubst %,$(OUT)/obj/%.o,$(SRC))
TOBJ := $(patsubst %,$(OUT)/obj/t_%.o,$(TESTS))

all: $(OUT)/libmidbf_ref.so $(OUT)/ref_unit_tests

$(OUT)/obj/%.o: $(REF)/src/%.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/obj/t_%.o: $(REF)/tests/%.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/obj/ref_capi.o: oracle/ref_capi.cpp $(SHIM)
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/libmidbf_ref.so: $(OBJ) $(OUT)/obj/ref_capi.o
	$(CXX) -shared -fopenmp -o $@ $^

$(OUT)/ref_unit_tests: $(TOBJ) $(OBJ)
	$(CXX) -fopenmp -o $@ $^ -Wl,--unresolved-symbols=ignore-all

clean:
	rm -rf $(OUT)

.PHONY: all clean
