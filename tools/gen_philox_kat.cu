// tools/gen_philox_kat.cu -- generates tests/golden/philox_kat.json from
// cuRAND's own Philox4x32-10 (curand_philox4x32_x.h:160-186), evaluated on the
// host.  The oracle (oracle/philox_ref.h) and the device engine are pinned to
// these vectors.  Build+run: nvcc -o /tmp/kat tools/gen_philox_kat.cu && /tmp/kat
#define QUALIFIERS static __forceinline__ __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
#include <cstdint>

int main() {
    const uint32_t cases[][6] = {
        {0u, 0u, 0u, 0u, 0u, 0u},
        {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu},
        {0x243f6a88u, 0x85a308d3u, 0x13198a2eu, 0x03707344u, 0xa4093822u, 0x299f31d0u},
        {1u, 2u, 3u, 4u, 5u, 6u},
        {123456789u, 0u, 77u, 0u, 0xdeadbeefu, 0x01234567u},
    };
    printf("{\n  \"source\": \"curand_Philox4x32_10 (CUDA 12.9 headers), host-evaluated\",\n  \"cases\": [\n");
    const int nc = sizeof(cases) / sizeof(cases[0]);
    for (int k = 0; k < nc; ++k) {
        uint4 c = make_uint4(cases[k][0], cases[k][1], cases[k][2], cases[k][3]);
        uint2 key = make_uint2(cases[k][4], cases[k][5]);
        uint4 o = curand_Philox4x32_10(c, key);
        printf("    {\"ctr\": [%u, %u, %u, %u], \"key\": [%u, %u], \"out\": [%u, %u, %u, %u]}%s\n",
               c.x, c.y, c.z, c.w, key.x, key.y, o.x, o.y, o.z, o.w, k + 1 < nc ? "," : "");
    }
    printf("  ]\n}\n");
    return 0;
}
