# Builds oracle/_ref/libigabem_ref.so: the REFERENCE's own core sources, read in
# place from /root/reference (never copied), compiled against the Eigen-subset
# shim in oracle/shim, plus the extern "C" harness.  Test infrastructure only.
CXX      := /usr/bin/g++
REF      := /root/reference/proj/core
CXXFLAGS := -std=c++20 -O2 -fPIC -fopenmp -ffp-contract=off -w -Ishim -I$(REF)/include -I$(REF)/src
SRCS     := splines quadrature geometry shapes spaces assembly h2 operators
OBJS     := $(addprefix _ref/,$(addsuffix .o,$(SRCS))) _ref/ref_harness.o

all: _ref/libigabem_ref.so
_ref:
	mkdir -p _ref
_ref/%.o: $(REF)/src/%.cpp shim/Eigen/Dense | _ref
	$(CXX) $(CXXFLAGS) -c $< -o $@
_ref/ref_harness.o: ref_harness.cpp shim/Eigen/Dense | _ref
	$(CXX) $(CXXFLAGS) -c $< -o $@
_ref/libigabem_ref.so: $(OBJS)
	$(CXX) -shared -fopenmp -o $@ $(OBJS)
clean:
	rm -rf _ref
.PHONY: all clean

# C++ drop-in test program: reference headers + shim + include/igabem_b200
../tests/cpp/dropin_test: ../tests/cpp/dropin_test.cpp ../include/igabem_b200/h2_dropin.hpp _ref/libigabem_ref.so
	$(CXX) $(CXXFLAGS) -I../include $< -o $@ -L_ref -ligabem_ref -L../paper_1906_00785_b200 -ligabem_b200 \
	  -Wl,-rpath,'$$ORIGIN/../../oracle/_ref' -Wl,-rpath,'$$ORIGIN/../../paper_1906_00785_b200'
all: ../tests/cpp/dropin_test
