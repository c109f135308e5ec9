# build a library variant with a different slot_fast.cu: sfvar.sh NAME SRC
set -e
cd /root/repo/paper_2506_14781_b200
cp $2 csrc/_sf_variant.cu
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -c csrc/_sf_variant.cu -o build/sf_$1.o
rm csrc/_sf_variant.cu
objs=$(ls build/*.o | grep -v "build/slot_fast.o" | grep -v "build/sf_" | grep -v "_[a-z0-9]*\.o$" )
objs="build/kernels.o build/capi.o build/host_common.o build/host_slot.o build/host_run.o build/host_extras.o build/host_ckpt.o build/plane_r0.o build/plane_r1.o build/tpw_r0.o build/tpw_r1.o build/plane_c5.o build/slot_engine.o build/prep.o build/host_plane.o"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libtempergrid_b200_$1.so $objs build/sf_$1.o -ldl
echo libtempergrid_b200_$1.so
