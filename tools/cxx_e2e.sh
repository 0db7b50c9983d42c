#!/bin/bash
# The plugin boundary timed from C++ on the reference's own types (oracle/_ref/ref_gpu_driver e2e, built where /root/reference
# exists): C4 and the n = 1e5 point, pageable std::vector genes -> profiles/<tag>_cxx_e2e.jsonl.  Test infrastructure, not bench.py.
TAG=${1:-r02e}
export GAPA_CUDA_LIB=$PWD/paper_2412_20980_b200/libgapa_cuda.so
: > gpurun_out/${TAG}_cxx_e2e.jsonl
oracle/_ref/ref_gpu_driver e2e 1000000 5 4096 5 | tail -1 >> gpurun_out/${TAG}_cxx_e2e.jsonl
oracle/_ref/ref_gpu_driver e2e 100000 5 4096 10 | tail -1 >> gpurun_out/${TAG}_cxx_e2e.jsonl
oracle/_ref/ref_gpu_driver e2e 10000 5 4096 20 | tail -1 >> gpurun_out/${TAG}_cxx_e2e.jsonl
cat gpurun_out/${TAG}_cxx_e2e.jsonl
