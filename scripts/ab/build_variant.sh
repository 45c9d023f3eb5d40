# build scripts/ab/libskp_<name>.so: the tree's objects with sketch_gather.cu recompiled with extra -D flags
# usage: bash scripts/ab/build_variant.sh NAME [-DFLAG ...]
set -e
name=$1; shift
P=paper_2605_09755_b200
python -m $P._build > /dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr -Xptxas -O3 -I include "$@" -c $P/csrc/sketch_gather.cu -o /tmp/sg_$name.o
objs=$(ls $P/build/*.o | grep -v sketch_gather.cu.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o scripts/ab/libskp_$name.so $objs /tmp/sg_$name.o -lcuda
echo built scripts/ab/libskp_$name.so
