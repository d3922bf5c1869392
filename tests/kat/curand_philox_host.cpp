// Independent Philox4x32-10 check: cuRAND's own curand_Philox4x32_10, compiled
// for the HOST (the header has a NV_IS_HOST branch for mulhilo32).  Reads lines
// "c0 c1 c2 c3 k0 k1" (decimal uint32) on stdin, prints "x0 x1 x2 x3".
// Test infrastructure for tests/test_oracle_noise.py (pins oracle/noise.py).
#define QUALIFIERS static inline
#include <cstdio>
#include <vector_types.h>
#include <curand_philox4x32_x.h>

int main() {
    unsigned c0, c1, c2, c3, k0, k1;
    while (std::scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
        uint4 c; c.x = c0; c.y = c1; c.z = c2; c.w = c3;
        uint2 k; k.x = k0; k.y = k1;
        uint4 r = curand_Philox4x32_10(c, k);
        std::printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
    }
    return 0;
}
