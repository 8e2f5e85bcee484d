# Builds the CUDA product library (sm_100a) and the C oracle (test infra).
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo --fmad=false -Xcompiler -fPIC,-Wall -shared -ldl
NVFLAGS   += $(NVEXTRA)
ifeq ($(WSPROF),1)
NVFLAGS   += -DKNNG_WS_PROF
endif
PKG       := paper_2103_15386_b200
LIB       := $(PKG)/lib/libknng.so
SRCS      := $(wildcard $(PKG)/csrc/*.cu $(PKG)/csrc/*.cuh) include/knng.h
ORACLE    := oracle/liboracle.so

all: $(LIB) $(ORACLE)

$(LIB): $(SRCS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -o $@ $(PKG)/csrc/knng_api.cu

$(ORACLE): oracle/knng_oracle.c oracle/knng_oracle.h
	gcc -std=gnu99 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -Wall -Wextra \
	    -Wno-unused-parameter -o $@ oracle/knng_oracle.c -lm

ptxas: $(SRCS)
	$(NVCC) $(NVFLAGS) -Xptxas -v -o /tmp/libknng_ptxas.so $(PKG)/csrc/knng_api.cu

clean:
	rm -f $(LIB) $(ORACLE)

.PHONY: all clean ptxas
