# timing probes of the cluster SAT step (wrong results by design): variant libraries built here, run on the box
set -e
cd "$(dirname "$0")/.."
L=paper_2012_11077_b200/lib
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-O2 -Iinclude"
mkdir -p $L/probe
for v in ${VARIANTS:-0 1 2 4 7}; do
  nvcc $F $EXTRA -DUWB_CL_PROBE=0 -DUWB_CL_SLACK=$v -c paper_2012_11077_b200/csrc/sat_cluster.cu -o $L/probe/sat_cluster_$v.o
  objs=$(ls $L/*.cu.o | grep -v sat_cluster)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared $objs $L/probe/sat_cluster_$v.o -o $L/probe/lib_$v.so
done
