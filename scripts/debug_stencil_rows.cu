// A/B of the band-edge stencil (k_edge_stencil) against k_stencil on the same random inputs (debug harness, one GPU):
// y and the reduction slots of the given rows must be bitwise equal, per precision mode.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "kernels.cuh"
using namespace eg;

// naive: slots from y and aux, serial k per column, 128 threads (k_stencil's CTA shape)
template <int MODE, int DOTS>
__global__ void k_naive(Geo g, Vecs<MODE> vv, const typename Prec<MODE>::V* y, const typename Prec<MODE>::V* aux,
                        RowMap rm) {
    using V = typename Prec<MODE>::V;
    constexpr int NQ = DOTS == 2 ? 3 : 1;
    double acc[NQ];
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    const int i = blockIdx.x * RW + threadIdx.x;
    const int64_t jl = rm.lo + (int64_t)blockIdx.y * rm.step;
    if (i < g.nx)
        for (int k = 0; k < g.nz; ++k) {
            const int64_t o = jl * g.row + (int64_t)k * g.nx + i;
            const V a = y[o], sv = aux[o];
            if (DOTS == 1) acc_dot<MODE>(acc[0], sv, a);
            else { acc_dot<MODE>(acc[0], a, sv); acc_dot<MODE>(acc[1], a, a); acc_dot<MODE>(acc[2], sv, sv); }
        }
    write_slots<NQ>(g, vv.slots, acc, MODE == 2 ? 0x7u : 0x0u, jl);
}

template <int MODE, int DOTS>
int run(int nx, int nyl, int nz) {
    using V = typename Prec<MODE>::V;
    Geo g{};
    g.nx = nx; g.ny = nyl; g.nz = nz; g.row = (int64_t)nx * nz; g.nyl = nyl; g.j0 = 0; g.n = g.row * nyl;
    g.tiles = (nx + RW - 1) / RW; g.G = 1; g.g_lo = 0; g.g_hi = 1; g.quad = 0;
    const int64_t n = g.n, row = g.row;
    std::vector<V> h4(4 * n), h2(2 * n), hz(n + 2 * row), ha(n);
    srand(7);
    auto rnd = [] { return (V)((rand() / (double)RAND_MAX) - 0.5); };
    for (auto& v : h4) v = rnd() * (V)0.2;
    for (auto& v : h2) v = rnd() * (V)0.2;
    for (auto& v : hz) v = rnd();
    for (auto& v : ha) v = rnd();
    V *b4, *b2, *z, *a, *y1, *y2; double *s1, *s2; DevState* st;
    cudaMalloc(&b4, 4 * n * sizeof(V)); cudaMalloc(&b2, 2 * n * sizeof(V)); cudaMalloc(&z, (n + 2 * row) * sizeof(V));
    cudaMalloc(&a, n * sizeof(V)); cudaMalloc(&y1, n * sizeof(V)); cudaMalloc(&y2, n * sizeof(V));
    cudaMalloc(&s1, 3 * nyl * g.tiles * 8); cudaMalloc(&s2, 3 * nyl * g.tiles * 8); cudaMalloc(&st, sizeof(DevState));
    cudaMemcpy(b4, h4.data(), 4 * n * sizeof(V), cudaMemcpyHostToDevice);
    cudaMemcpy(b2, h2.data(), 2 * n * sizeof(V), cudaMemcpyHostToDevice);
    cudaMemcpy(z, hz.data(), (n + 2 * row) * sizeof(V), cudaMemcpyHostToDevice);
    cudaMemcpy(a, ha.data(), n * sizeof(V), cudaMemcpyHostToDevice);
    cudaMemset(st, 0, sizeof(DevState));
    cudaMemset(s1, 0, 3 * nyl * g.tiles * 8); cudaMemset(s2, 0, 3 * nyl * g.tiles * 8);
    Vecs<MODE> vv{};
    vv.B4 = b4; vv.B2 = b2; vv.st = st;
    RowMap rm{0, nyl - 1};
    const int nr = nyl > 1 ? 2 : 1;
    vv.slots = s1;
    k_stencil<MODE, DOTS><<<dim3(g.tiles, nr), RW>>>(g, vv, z + row, y1, a, rm);
    vv.slots = s2;
    int* ctr; cudaMalloc(&ctr, 2 * g.tiles * 4); cudaMemset(ctr, 0, 2 * g.tiles * 4);
    cudaFuncSetAttribute(k_edge_stencil<MODE, DOTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)es_smem_bytes<MODE>());
    k_edge_stencil<MODE, DOTS><<<dim3(g.tiles, nr, (nz + 3) / 4), 512, es_smem_bytes<MODE>()>>>(g, vv, z + row, y2, a, rm,
                                                                                              HWait{nullptr, 0, 0, 0, 0}, ctr, nullptr);
    double* s3; cudaMalloc(&s3, 3 * nyl * g.tiles * 8); cudaMemset(s3, 0, 3 * nyl * g.tiles * 8);
    vv.slots = s3;
    k_naive<MODE, DOTS><<<dim3(g.tiles, nr), RW>>>(g, vv, y1, a, rm);
    cudaDeviceSynchronize();
    std::vector<double> q3(3 * nyl * g.tiles);
    cudaMemcpy(q3.data(), s3, q3.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<V> o1(n), o2(n);
    std::vector<double> q1(3 * nyl * g.tiles), q2(3 * nyl * g.tiles);
    cudaMemcpy(o1.data(), y1, n * sizeof(V), cudaMemcpyDeviceToHost);
    cudaMemcpy(o2.data(), y2, n * sizeof(V), cudaMemcpyDeviceToHost);
    cudaMemcpy(q1.data(), s1, q1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(q2.data(), s2, q2.size() * 8, cudaMemcpyDeviceToHost);
    int by = 0, bs = 0;
    for (int j : {0, nyl - 1})
        for (int64_t q = j * row; q < (j + 1) * row; ++q) by += o1[q] != o2[q];
    for (size_t q = 0; q < q1.size(); ++q)
        if (q1[q] != q2[q]) { if (bs < 4) printf("   slot %zu: %.17g vs %.17g\n", q, q1[q], q2[q]); ++bs; }
    int b13 = 0, b23 = 0;
    for (size_t q = 0; q < q1.size(); ++q) { b13 += q1[q] != q3[q]; b23 += q2[q] != q3[q]; }
    printf("   vs naive: k_stencil %d, edge kernels %d\n", b13, b23);
    printf("MODE %d DOTS %d %dx%dx%d: y mismatches %d, slot mismatches %d (%s)\n", MODE, DOTS, nx, nyl, nz, by, bs,
           cudaGetErrorString(cudaGetLastError()));
    return by + bs;
}
int main() {
    int bad = 0;
    for (int nz : {13, 70}) {
        bad += run<0, 1>(200, 9, nz); bad += run<0, 2>(200, 9, nz);
        bad += run<1, 1>(200, 9, nz); bad += run<1, 2>(200, 9, nz);
        bad += run<2, 1>(200, 9, nz); bad += run<2, 2>(200, 9, nz);
    }
    printf("%s\n", bad ? "MISMATCH" : "all equal");
    return bad != 0;
}
