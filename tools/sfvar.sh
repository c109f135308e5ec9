# build a library variant that differs in slot_fast.cu's compile flags: tools/sfvar.sh NAME "-DTG_SF_...=0"
# -> paper_2506_14781_b200/libtempergrid_b200_NAME.so (select with TG_ENGINE_LIB; tools/abfloat.sh NAME...)
set -e
cd "$(dirname "$0")/../paper_2506_14781_b200"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC $2 -c csrc/slot_fast.cu -o build/sf_$1.o
objs="build/kernels.o build/capi.o build/host_common.o build/host_slot.o build/host_run.o build/host_extras.o build/host_ckpt.o build/plane_r0.o build/plane_r1.o build/tpw_r0.o build/tpw_r1.o build/plane_c5.o build/plane_cl.o build/slot_engine.o build/prep.o build/host_plane.o"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libtempergrid_b200_$1.so $objs build/sf_$1.o -ldl
echo libtempergrid_b200_$1.so
