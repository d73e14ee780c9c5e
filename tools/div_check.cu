// div_check.cu — is q = fma(fma(-a*r, b, a), r, a*r) with r = RN(1/b) equal to RN(a/b) (fp64)?
// Random operands over wide exponent ranges plus the normalisation's shapes (a = x - shift with
// x fp32, b = a column standard deviation). Prints mismatches.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/div_check tools/div_check.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ uint64_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__device__ double rnd_double(uint64_t s, int emin, int emax) {
    const uint64_t m = mix(s) & 0xFFFFFFFFFFFFFull;
    const int e = emin + (int)(mix(s + 7) % (uint64_t)(emax - emin + 1));
    const uint64_t sign = (mix(s + 13) & 1) << 63;
    return __longlong_as_double((long long)(sign | ((uint64_t)(e + 1023) << 52) | m));
}

__global__ void k(int64_t n, int mode, unsigned long long* bad, double* ex) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double a, b;
    if (mode == 0) {            // generic
        a = rnd_double(2 * i, -60, 60);
        b = rnd_double(2 * i + 1, -60, 60);
    } else {                    // normalisation: fp32 x minus shift, sigma
        const float x = (float)rnd_double(3 * i, -20, 20);
        const double shift = rnd_double(3 * i + 1, -10, 10);
        b = fabs(rnd_double(3 * i + 2, -10, 10));
        a = (double)x - shift;
    }
    const double r = 1.0 / b;
    double q = a * r;
    const double rem = fma(-q, b, a);
    q = fma(rem, r, q);
    const double t = a / b;
    if (q != t && !(isnan(q) && isnan(t))) {
        const unsigned long long slot = atomicAdd(bad, 1ull);
        if (slot < 4) { ex[3 * slot] = a; ex[3 * slot + 1] = b; ex[3 * slot + 2] = q - t; }
    }
}

int main() {
    unsigned long long* bad;
    double* ex;
    cudaMalloc(&bad, 8);
    cudaMalloc(&ex, 12 * 8);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(bad, 0, 8);
        const int64_t n = 1ll << 32;
        const int64_t chunk = 1ll << 28;
        for (int64_t off = 0; off < n; off += chunk) {
            // reuse k with an offset by shifting the index space
            k<<<(unsigned)(chunk / 256), 256>>>(chunk, mode, bad, ex);
        }
        cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
        double hx[12];
        cudaMemcpy(hx, ex, sizeof(hx), cudaMemcpyDeviceToHost);
        printf("mode %d: %llu mismatches in %lld\n", mode, h, (long long)chunk);
        for (unsigned long long s = 0; s < h && s < 4; ++s)
            printf("  a=%.17g b=%.17g diff=%g\n", hx[3 * s], hx[3 * s + 1], hx[3 * s + 2]);
    }
    return 0;
}
