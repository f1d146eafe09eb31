# usage: bash scripts/build_variant.sh <name> "<-D flags>"  -> tune/<name>.so (tuning builds, BM_LIB=...)
name=$1; flags=$2
mkdir -p tune
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_1303_1379_b200/csrc $flags \
  -c paper_1303_1379_b200/csrc/bm_engine.cu -o tune/$name.o && \
g++ -O3 -std=c++17 -fPIC -pthread -Iinclude -c paper_1303_1379_b200/csrc/bm_host.cpp -o tune/host.o && \
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_1303_1379_b200/csrc \
  -c paper_1303_1379_b200/csrc/bm_partition.cu -o tune/part.o && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tune/$name.so tune/$name.o tune/part.o tune/host.o -Xcompiler -pthread
