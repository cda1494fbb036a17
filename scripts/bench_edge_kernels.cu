// In-pipeline cost of the band-edge kernels at a band's shape (default: the C4 band of P = 8,
// 1536 x 144 x 70, fp32 working precision): each kernel launched back to back 400 times on one
// stream, CUDA events around the loop (the GPU stays busy, so it runs at its load clock — ncu's
// serialised replay leaves it idling between tiny kernels).  k_stencil over the two edge rows (the
// round-1 column walk) is timed beside the two-kernel edge stencil that replaced it.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "kernels.cuh"
using namespace eg;

int main(int argc, char** argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 1536, nyl = argc > 2 ? atoi(argv[2]) : 144, nz = argc > 3 ? atoi(argv[3]) : 70;
    constexpr int MODE = 1;
    using V = float;
    Geo g{};
    g.nx = nx; g.ny = 8 * nyl; g.nz = nz; g.row = (int64_t)nx * nz; g.nyl = nyl; g.j0 = 3 * nyl; g.n = g.row * nyl;
    g.tiles = (nx + RW - 1) / RW; g.G = 8; g.g_lo = 3; g.g_hi = 4; g.quad = 0;
    const int64_t n = g.n, row = g.row;
    auto alloc = [](size_t b) { void* p; cudaMalloc(&p, b); cudaMemset(p, 0, b); return p; };
    std::vector<float> h(6 * n);
    for (auto& v : h) v = (float)(rand() / (double)RAND_MAX) * 0.1f;
    Vecs<MODE> vv{};
    V* b4 = (V*)alloc(4 * n * 4); V* b2 = (V*)alloc(2 * n * 4);
    cudaMemcpy(b4, h.data(), 4 * n * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(b2, h.data(), 2 * n * 4, cudaMemcpyHostToDevice);
    vv.B4 = b4; vv.B2 = b2;
    vv.r = (V*)alloc(n * 4); vv.rh = (V*)alloc(n * 4); vv.p = (V*)alloc(n * 4); vv.v = (V*)alloc(n * 4);
    vv.s = (V*)alloc(n * 4); vv.t = (V*)alloc(n * 4);
    cudaMemcpy(vv.r, h.data(), n * 4, cudaMemcpyHostToDevice);
    V* zext = (V*)alloc((n + 2 * row) * 4);
    cudaMemcpy(zext, h.data(), (n + 2 * row) * 4, cudaMemcpyHostToDevice);
    vv.z = zext + row;
    vv.slots = (double*)alloc(3 * nyl * g.tiles * 8);
    DevState* st = (DevState*)alloc(sizeof(DevState));
    vv.st = st;
    float* scratch = (float*)alloc(2 * row * 4);
    P2P pp{};
    const size_t ers = er_smem_bytes(nz);
    cudaFuncSetAttribute(k_edge_rows<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ers);
    cudaFuncSetAttribute(k_edge_rows<MODE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ers);
    RowMap rm{0, nyl - 1};
    const dim3 ge((nx + ER_COLS - 1) / ER_COLS, 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto&& launch) {
        for (int w = 0; w < 20; ++w) launch();
        cudaEventRecord(e0);
        for (int it = 0; it < 400; ++it) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-44s %8.2f us per launch (%s)\n", name, 1000.f * ms / 400, cudaGetErrorString(cudaGetLastError()));
    };
    printf("band %d x %d x %d (fp32 V)\n", nx, nyl, nz);
    timeit("k_edge_rows<1> (z, staged)", [&] { k_edge_rows<MODE, 1><<<ge, ER_THREADS, ers>>>(g, vv, scratch, pp, nullptr); });
    timeit("k_edge_rows<2> (z_s, staged)", [&] { k_edge_rows<MODE, 2><<<ge, ER_THREADS, ers>>>(g, vv, scratch, pp, nullptr); });
    timeit("k_stencil<1> on the 2 edge rows (column walk)",
           [&] { k_stencil<MODE, 1><<<dim3(g.tiles, 2), RW>>>(g, vv, vv.z, vv.v, vv.rh, rm); });
    int* ctr = (int*)alloc(2 * g.tiles * 4);
    const size_t ess = es_smem_bytes<MODE>();
    cudaFuncSetAttribute(k_edge_stencil<MODE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ess);
    cudaFuncSetAttribute(k_edge_stencil<MODE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ess);
    cudaFuncSetAttribute(k_edge_stencil<MODE, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ess);
    timeit("k_edge_stencil<1>", [&] {
        k_edge_stencil<MODE, 1><<<dim3(g.tiles, 2, (nz + 3) / 4), 512, ess>>>(g, vv, vv.z, vv.v, vv.rh, rm, HWait{nullptr, 0, 0, 0, 0}, ctr, nullptr);
    });
    timeit("k_edge_stencil<0> (points only)", [&] {
        k_edge_stencil<MODE, 0><<<dim3(g.tiles, 2, (nz + 3) / 4), 512, ess>>>(g, vv, vv.z, vv.v, vv.rh, rm, HWait{nullptr, 0, 0, 0, 0}, ctr, nullptr);
    });
    timeit("k_stencil<2> on the 2 edge rows (column walk)",
           [&] { k_stencil<MODE, 2><<<dim3(g.tiles, 2), RW>>>(g, vv, vv.zs = vv.z, vv.t, vv.s, rm); });
    timeit("k_edge_stencil<2>", [&] {
        k_edge_stencil<MODE, 2><<<dim3(g.tiles, 2, (nz + 3) / 4), 512, ess>>>(g, vv, vv.z, vv.t, vv.s, rm, HWait{nullptr, 0, 0, 0, 0}, ctr, nullptr);
    });
    timeit("k_copy-like empty kernel (1 CTA, launch floor)", [&] { k_edge_stencil<MODE, 0><<<dim3(1, 1, 1), 32, ess>>>(g, vv, vv.z, vv.v, vv.rh, RowMap{0, 0}, HWait{nullptr, 0, 0, 0, 0}, ctr, nullptr); });
    return 0;
}
