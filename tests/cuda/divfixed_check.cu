// Device check of pp::div_fixed / pp::div_recip against the compiler's IEEE
// division, bit for bit (tests/test_gpu_divfixed.py builds and runs it).
#include "../../paper_2204_10562_b200/csrc/common.cuh"

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// a random double of one of several shapes: random mantissa, all-ones mantissa,
// power of two, small integer; exponent drawn over the whole range or near 1
__device__ double draw(unsigned long long h) {
    const unsigned kind = h & 7, wide = (h >> 3) & 3;
    unsigned long long m = mix(h) & 0xfffffffffffffULL;
    if (kind == 1) m = 0xfffffffffffffULL;
    if (kind == 2) m = 0;
    if (kind == 3) m = (mix(h) & 0xfULL) << 48;
    if (kind == 4) return (double)((h >> 8) % 1000 + 1);
    const unsigned e = wide == 0 ? 1 + (unsigned)((h >> 8) % 2046) : 1023 - 40 + (unsigned)((h >> 8) % 80);
    return __longlong_as_double((long long)(((unsigned long long)e << 52) | m));
}

extern "C" __global__ void k_divfixed(unsigned long long seed, long long n, unsigned long long* bad, int per_b) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const double b = draw(mix(seed ^ (unsigned long long)t * 0x632be59bd9b4e019ULL));
        const double y = pp::div_recip(b);
        const bool ok = pp::div_fixed_ok(b);
        for (int k = 0; k < per_b; ++k) {
            const double a = draw(mix(seed + 0x1234567ULL * (unsigned long long)(t * per_b + k + 1)));
            const double want = a / b, got = pp::div_fixed(a, b, y, ok);
            if (__double_as_longlong(want) != __double_as_longlong(got)) {
                const unsigned long long c = atomicAdd(&bad[0], 1ULL);
                if (c < 4) { bad[1 + 2 * c] = __double_as_longlong(a); bad[2 + 2 * c] = __double_as_longlong(b); }
            }
        }
    }
}

// host entry: n divisors x per_b numerators; returns the mismatch count and up
// to 4 (a, b) bit patterns in out[1..8]
extern "C" int run_divfixed(unsigned long long seed, long long n, int per_b, unsigned long long* out) {
    unsigned long long* d = nullptr;
    if (cudaMalloc(&d, 9 * sizeof(unsigned long long)) != cudaSuccess) return -1;
    cudaMemset(d, 0, 9 * sizeof(unsigned long long));
    k_divfixed<<<148 * 8, 256>>>(seed, n, d, per_b);
    const cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out, d, 9 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? 0 : -2;
}
