// Check: ddiv_fast (fvv_device.cuh) == __ddiv_rn on the blend's operand domain.
// Two kernels (so the compiler cannot merge the two divisions) fold the bit
// patterns of their quotients into per-thread hashes that are then compared.
#include <cstdio>
#include <cstdint>
#include "../../paper_2112_10603_b200/csrc/fvv_device.cuh"
using namespace fvv;
template <bool FAST>
__global__ void k(unsigned long long seed, int iters, double eps, unsigned long long* hash) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long s = seed ^ (0x9E3779B97F4A7C15ull * (tid + 1));
    unsigned long long h = 0;
    for (int i = 0; i < iters; i++) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        const double D = (double)(s & 0xFFFFFFF) / (double)(1 << 20);          // [0, 256)
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        const float ol = (float)((s >> 8) & 0xFFFFFF) / (float)(1 << 14);     // [0, 1024)
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        const float orr = (i & 3) == 0 ? 0.0f : (float)((s >> 8) & 0xFFFFFF) / (float)(1 << 14);
        const float ql = __fadd_rn(0.5f, __fmul_rn(4.0f, ol)), qr = __fadd_rn(0.5f, __fmul_rn(4.0f, orr));
        const double Dz = (i & 7) == 1 ? 0.0 : D;
        const double el = __dmul_rn(Dz, (double)ql), er = __dmul_rn(Dz, (double)qr);
        const double n = __dadd_rn(er, eps), d = __dadd_rn(__dadd_rn(el, er), 2.0 * eps);
        const double q = FAST ? ddiv_fast(n, d) : __ddiv_rn(n, d);
        h = (h * 0x100000001B3ull) ^ (unsigned long long)__double_as_longlong(q);
    }
    hash[tid] = h;
}
int main() {
    const int nb = 148 * 8, nt = 256, n = nb * nt, iters = 2000;
    unsigned long long *ha, *hb;
    cudaMallocManaged(&ha, 8ull * n);
    cudaMallocManaged(&hb, 8ull * n);
    const double epss[] = {1e-3, 1e-30, 1e-12, 0.5, 1e30};
    int fails = 0;
    for (double eps : epss) {
        k<false><<<nb, nt>>>(12345, iters, eps, ha);
        k<true><<<nb, nt>>>(12345, iters, eps, hb);
        cudaDeviceSynchronize();
        int bad = 0;
        for (int i = 0; i < n; i++) bad += ha[i] != hb[i];
        printf("eps %g: %d of %d thread hashes differ (%lld quotients)\n", eps, bad, n, (long long)n * iters);
        fails += bad != 0;
    }
    printf(fails ? "FAIL\n" : "OK\n");
    return fails;
}
