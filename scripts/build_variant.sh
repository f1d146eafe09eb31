# usage: bash scripts/build_variant.sh <name> "<-D flags>"  -> tunelib/<name>.so (tuning builds, selected with BM_LIB=...)
name=$1; flags=$2
mkdir -p tunelib
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_1303_1379_b200/csrc"
$NV $flags -c paper_1303_1379_b200/csrc/bm_engine.cu -o tunelib/$name.o && \
g++ -O3 -std=c++17 -fPIC -pthread -Iinclude -c paper_1303_1379_b200/csrc/bm_host.cpp -o tunelib/host.o && \
g++ -O3 -std=c++17 -fPIC -pthread -Iinclude -c paper_1303_1379_b200/csrc/bm_io.cpp -o tunelib/io.o && \
$NV $flags -c paper_1303_1379_b200/csrc/bm_mg.cu -o tunelib/mg_$name.o && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tunelib/$name.so tunelib/$name.o tunelib/mg_$name.o tunelib/host.o tunelib/io.o -Xcompiler -pthread && \
rm -f tunelib/$name.o tunelib/mg_$name.o
