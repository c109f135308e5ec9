# Build an engine variant that differs only in the PLANE kernels' compile flags
# (plane_tpw.cu, plane_c5.cu, plane_cl.cu, host_plane.cu):
#   tools/variant.sh NAME "-DTG_MULWIDE=1 ..."
# -> paper_2506_14781_b200/libtempergrid_b200_NAME.so (select with TG_ENGINE_LIB)
set -e
cd "$(dirname "$0")/../paper_2506_14781_b200"
NV="nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC"
for r in 0 1; do $NV -DTG_PLANE_RULE=$r $2 -c csrc/plane_tpw.cu -o build/tpw_r${r}_$1.o & done
$NV $2 -c csrc/plane_c5.cu -o build/plane_c5_$1.o &
$NV $2 -c csrc/plane_cl.cu -o build/plane_cl_$1.o &
$NV $2 -c csrc/host_plane.cu -o build/host_plane_$1.o &
wait
objs="build/kernels.o build/capi.o build/host_common.o build/host_slot.o build/host_run.o build/host_extras.o build/host_ckpt.o build/plane_r0.o build/plane_r1.o build/slot_engine.o build/slot_fast.o build/prep.o"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libtempergrid_b200_$1.so $objs build/tpw_r0_$1.o build/tpw_r1_$1.o build/plane_c5_$1.o build/plane_cl_$1.o build/host_plane_$1.o -ldl
echo libtempergrid_b200_$1.so
