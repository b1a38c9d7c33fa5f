#!/bin/bash
# Rebuild the in-tree library with the sweep's phase timers (-DDM_MITM_TIMING);
# `make -C paper_2309_01172_b200/csrc` afterwards restores the normal build.
set -e
cd "$(dirname "$0")/../../paper_2309_01172_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC,-fvisibility=hidden \
     -DDM_MITM_TIMING -c -o /tmp/dm_mitm_t.o dm_mitm.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libdagmesh_b200.so dm_eval.o dm_enum.o /tmp/dm_mitm_t.o \
     dm_dp.o dm_hill.o dm_peak.o dm_opcost.o dm_random.o dm_sched.o
touch dm_mitm.cu
