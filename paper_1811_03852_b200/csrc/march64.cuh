// march64.cuh — fused phase kernels of the BiCGStab iteration in the all-fp64 variant (EG_FP64,
// Table 1's "DP" column).  Same schedule as march.cuh (read it first):
//
//   phase A (rows a3 + a4):  p = r + beta (p - omega v);  z = T^-1 p;  v = Ahat z;  partial rhat0 . v
//   phase B (rows a6 + a7):  s = r - alpha v;  z_s = T^-1 s;  t = Ahat z_s;  partials t.s, t.t, s.s
//
// one persistent CTA per SM marches a tile of a latitude strip row by row: the Thomas warps (F)
// eliminate and back-substitute row r_{m+2} into a 3-row shared-memory z ring while the stencil
// warps (S) apply the operator to row r_m.  What changes with 8-byte values:
//   * tiles are 64 columns wide: a 3-row fp64 z ring of 128 columns (224 KB) does not fit the 227 KB
//     of shared memory; with 64 it is 114 KB.  Two F and two S warps (TMEM lanes 0-63);
//   * TMEM holds c' (word pairs, 2 NZ4 columns) and, in phase B, s of two rows (4 NZ4): <= 432 of
//     512 columns at nz = 70.  The (U, D) bands of the stencil row do NOT fit next to them (they
//     would need 4 NZ4 more), so the stencil producer streams them again with its (E, W, N, S) box:
//     the elimination read them two rows earlier, so the second read is normally an L2 hit;
//   * chunks are one 4-level stage (KB = KS = 4), the register budget of fp64.
// Algorithmic HBM bytes per point: phase A 104 (r, p, v, rhat0, 6 bands in; p, z, v out), phase B
// 88 (r, v, 6 bands in; s, z_s, t out); with the 64 B update, 256 B per iteration.
//
// Arithmetic, operation for operation, is k_thomas / k_thomas_tma64 (division for 1/m, the
// explicit z_{nz-1} = y_{nz-1}) and k_stencil<0>, so the fused FP64 schedule is bitwise identical to
// the 5-kernel one.  The dot-product partials are the 5-kernel's too: k_stencil sums a 128-column
// slot as ((w0 + w1) + w2) + w3 over its four warps; a 64-column CTA writes its two warp sums to
// half-slots (hslots[q][row][tile][4]) and the finaliser forms the same sum (Geo.quad).
// Requires nx % 2 == 0 (16-byte TMA strides), 6 * ceil4(nz) <= 512, ceil(nx/64) tiles <= #SMs; one
// GPU (latitude bands run the 5-kernel FP64 schedule).
#pragma once
#include "sor_tma.cuh"

namespace eg {

constexpr int M6_KS = 4;                          // levels per stage = per chunk
constexpr int M6_TILE = 64;                       // columns per CTA
constexpr int M6_CONS = 64;                       // consumer threads per role
constexpr int M6_THREADS = 256;                   // S 0-1, producers 2-3, F 4-5, publisher 6, halo 7
constexpr int M6_RING_W = M6_TILE + 2;            // W halo | 64 columns | E halo
constexpr int M6_MAX_NZ4 = 84;                    // 6 * 84 = 504 TMEM columns
constexpr int M6_MAX_CH = M6_MAX_NZ4 / M6_KS;
constexpr int M6_MAX_STAGES = 16;
// stage layouts (doubles).  Elimination: r | (p |) v | (U, D).  Stencil: (E, W, N, S) | (rhat0 |) (U, D)
constexpr int m6_f_doubles(int kind) { return M6_KS * M6_TILE * (kind == 1 ? 5 : 4); }
constexpr int m6_s_doubles(int kind) { return M6_KS * M6_TILE * (kind == 1 ? 7 : 6); }
constexpr int m6_f_bytes(int kind) { return 8 * m6_f_doubles(kind); }
constexpr int m6_s_bytes(int kind) { return 8 * m6_s_doubles(kind); }
constexpr uint32_t M6_BOX_V = M6_KS * M6_TILE * 8;   // one fp64 array
constexpr uint32_t M6_BOX_B2 = 2 * M6_BOX_V;
constexpr uint32_t M6_BOX_B4 = 4 * M6_BOX_V;

// [nyl][nz][nx] views with 64 x KS boxes; (U, D) and (E, W, N, S) as 8-byte elements of [nyl][nz][2nx]
// (128 x KS boxes) and [nyl][nz][4nx] (256 x KS boxes)
struct MarchMaps64 {
    CUtensorMap r, p, v, rh, b2, b4;
};

__device__ __forceinline__ void tm_st8d(uint32_t taddr, const double (&d)[4]) {
    float w[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) split_d(d[e], w[2 * e], w[2 * e + 1]);
    tm_st8(taddr, w);
}
__device__ __forceinline__ void cons6_bar() { asm volatile("bar.sync 1, 64;" ::: "memory"); }

template <int KIND>
__global__ void __launch_bounds__(M6_THREADS, 1) k_march64(Geo g, Vecs<0> vv, MarchGeo mg, int* __restrict__ flags,
                                                           double* __restrict__ hslots,
                                                           const __grid_constant__ MarchMaps64 maps) {
    using V = double;
    constexpr int KS = M6_KS;
    constexpr int TW = M6_TILE;
    constexpr int SFD = m6_f_doubles(KIND), SSD = m6_s_doubles(KIND);
    constexpr int F_P = KS * TW;                              // p after r (phase A)
    constexpr int F_V = (KIND == 1 ? 2 : 1) * KS * TW;       // v after r (, p)
    constexpr int F_UD = (KIND == 1 ? 3 : 2) * KS * TW;      // (U, D) after r, (p,) v
    constexpr int S_RH = 4 * KS * TW;                         // rhat0 after (E, W, N, S)
    constexpr int S_UD = (KIND == 1 ? 5 : 4) * KS * TW;      // (U, D) after (E, W, N, S) (, rhat0)
    extern __shared__ __align__(128) unsigned char smtma[];
    __shared__ __align__(8) uint64_t fullF[M6_MAX_STAGES], emptyF[M6_MAX_STAGES];
    __shared__ __align__(8) uint64_t fullS[M6_MAX_STAGES], emptyS[M6_MAX_STAGES];
    __shared__ __align__(8) uint64_t sread[M6_MAX_CH], zready[2], zdone[2];
    __shared__ __align__(8) uint64_t hready[2], hfree[2], pubd[2];
    __shared__ double hbuf[2][2][M6_MAX_NZ4];  // E / W halo columns of rows r_x, slot x & 1
    __shared__ uint32_t tm_slot;
    DevState* st = vv.st;
    if (st->halt != H_RUN) return;  // uniform
    const int epoch = st->epoch;
    const bool fresh = KIND == 1 && st->fresh != 0;
    V beta = 0.0, omega = 0.0, alpha = 0.0;
    if (KIND == 1) {
        beta = st->beta_v;
        omega = st->omega_v;
    } else {
        alpha = st->alpha_v;
    }
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nx = (int)g.nx, nz = (int)g.nz, nyl = (int)g.nyl;
    const int T = (nx + TW - 1) / TW;  // 64-column tiles
    const int NSF = KIND == 1 ? mg.fst_a : mg.fst_b, NSS = KIND == 1 ? mg.sst_a : mg.sst_b;
    const int t = blockIdx.x % T, strip = blockIdx.x / T;
    const int ja = (int)((int64_t)strip * nyl / mg.strips), jb = (int)((int64_t)(strip + 1) * nyl / mg.strips);
    const int L = jb - ja;
    const int dir = (strip & 1) ? -1 : 1;
    const int rfirst = dir > 0 ? ja : jb - 1;
    const int i0 = t * TW;
    const int w = min(TW, nx - i0);  // columns of this tile (even)
    const int nch = (nz + KS - 1) / KS;
    const int NZ4 = nch * KS;
    V* stF = reinterpret_cast<V*>(smtma + ((128u - (smem_u32(smtma) & 127u)) & 127u));
    V* stS = stF + (size_t)NSF * SFD;
    V* ring = stS + (size_t)NSS * SSD;  // [3][NZ4][66]
    const int ring_slot = NZ4 * M6_RING_W;

    if (tid == 0) {
        for (int s = 0; s < NSF; ++s) { mbar_init(&fullF[s], 1); mbar_init(&emptyF[s], M6_CONS); }
        for (int s = 0; s < NSS; ++s) { mbar_init(&fullS[s], 1); mbar_init(&emptyS[s], M6_CONS); }
        for (int c = 0; c < M6_MAX_CH; ++c) mbar_init(&sread[c], M6_CONS);
        for (int b = 0; b < 2; ++b) { mbar_init(&zready[b], M6_CONS); mbar_init(&zdone[b], M6_CONS); }
        for (int b = 0; b < 2; ++b) { mbar_init(&hready[b], 32); mbar_init(&hfree[b], M6_CONS); mbar_init(&pubd[b], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint32_t tbase = tm_alloc512(&tm_slot);  // contains __syncthreads()
    auto row_of = [&](int n) { return rfirst + dir * n; };

    // ------------------------------------------------------------------ producer warps
    if (warp == 2 || warp == 3) {
        if (lane == 0 && L > 0) {
            int fslot = 0, fround = 0, sslot = 0, sround = 0;
            auto fwd_stage = [&](int jr, int k0) {
                if (fround > 0) mbar_wait_sleep(&emptyF[fslot], (uint32_t)((fround - 1) & 1), 32);
                uint64_t* fb = &fullF[fslot];
                mbar_expect_tx(fb, (KIND == 1 ? (fresh ? 1u : 3u) : 2u) * M6_BOX_V + M6_BOX_B2);
                V* sb = stF + (size_t)fslot * SFD;
                tma3(sb, &maps.r, i0, k0, jr, fb);
                if (KIND == 1 && !fresh) tma3(sb + F_P, &maps.p, i0, k0, jr, fb);
                if (KIND == 2 || !fresh) tma3(sb + F_V, &maps.v, i0, k0, jr, fb);
                tma3(sb + F_UD, &maps.b2, 2 * i0, k0, jr, fb);
                if (++fslot == NSF) { fslot = 0; ++fround; }
            };
            auto sten_stage = [&](int jr, int k0) {
                if (sround > 0) mbar_wait_sleep(&emptyS[sslot], (uint32_t)((sround - 1) & 1), 32);
                uint64_t* fb = &fullS[sslot];
                mbar_expect_tx(fb, M6_BOX_B4 + M6_BOX_B2 + (KIND == 1 ? M6_BOX_V : 0u));
                V* sb = stS + (size_t)sslot * SSD;
                tma3(sb, &maps.b4, 4 * i0, k0, jr, fb);
                if (KIND == 1) tma3(sb + S_RH, &maps.rh, i0, k0, jr, fb);
                tma3(sb + S_UD, &maps.b2, 2 * i0, k0, jr, fb);
                if (++sslot == NSS) { sslot = 0; ++sround; }
            };
            for (int m = 0; m < L; ++m)
                for (int k0 = 0; k0 < NZ4; k0 += KS) {
                    if (warp == 2) fwd_stage(row_of(m), k0);
                    else sten_stage(row_of(m), k0);
                }
        }
        return;  // the compute warps keep the CTA (and its TMEM) alive until every stage has landed
    }
    // ------------------------------------------------------------------ publisher warp
    if (warp == 6) {
        if (lane == 0)
            for (int x = 0; x < L; ++x) {
                mbar_wait_sleep(&zdone[x & 1], (uint32_t)((x >> 1) & 1), 256);
                st_release(flags + (int64_t)row_of(x) * T + t, epoch);  // gpu-scope release: z(r_x)
                mbar_arrive(&pubd[x & 1]);
            }
        return;
    }
    // ------------------------------------------------------------------ halo warp
    const int tW = (t == 0) ? T - 1 : t - 1, tE = (t + 1 == T) ? 0 : t + 1;
    const int iWg = (i0 == 0) ? nx - 1 : i0 - 1;
    const int iEg = (i0 + w == nx) ? 0 : i0 + w;
    if (warp == 7) {
        V* __restrict__ Zh = KIND == 1 ? vv.z : vv.zs;
        for (int x = 0; x < L; ++x) {
            if (x >= 2) mbar_wait_sleep(&hfree[x & 1], (uint32_t)(((x - 2) >> 1) & 1), 64);
            const int jr = row_of(x);
            if (lane < 2) {
                const int* f = flags + (int64_t)jr * T + (lane == 0 ? tW : tE);
                while (ld_acquire(f) != epoch) __nanosleep(64);
            }
            __syncwarp();
            for (int k = lane; k < nz; k += 32) {
                const V* zg = Zh + (int64_t)jr * g.row + (int64_t)k * nx;
                hbuf[x & 1][0][k] = __ldcg(zg + iWg);
                hbuf[x & 1][1][k] = __ldcg(zg + iEg);
            }
            mbar_arrive(&hready[x & 1]);
        }
        return;
    }

    // ------------------------------------------------------------------ compute warps (S and F)
    const bool isF = warp >= 4;
    const int col = tid & 63;
    const bool act = col < w;
    const bool uni = w == TW;
    const int i = i0 + (act ? col : w - 1);  // inactive lanes compute on zero-filled data, never store
    const uint32_t tl = tbase + ((uint32_t)((warp & 1) * 32) << 16);
    // TMEM column map (per lane = per column, 32-bit words): c' [0, 2 NZ4) | s slots [2 NZ4, 6 NZ4)
    auto tS = [&](int slot) { return tl + (uint32_t)(2 * NZ4 + slot * 2 * NZ4); };
    V* __restrict__ Zw = KIND == 1 ? vv.z : vv.zs;
    auto slot_ptr = [&](int x) { return ring + (size_t)(((x % 3) + 3) % 3) * ring_slot; };

    if (isF) {
        // ============================ Thomas warps ============================
        V* __restrict__ Pw = KIND == 1 ? vv.p : vv.s;
        int cslot = 0;
        uint32_t cphase = 0;
        V cprev = 0.0, yprev = 0.0;
        auto fwd_chunk = [&](int k0, int c, V* zr, V* pw, int us, int sync_step) {
            V rr[KS], pp[KS], vq[KS], uu[KS], dd[KS];
            mbar_wait(&fullF[cslot], cphase);
            const V* sb = stF + (size_t)cslot * SFD;
#pragma unroll
            for (int l = 0; l < KS; ++l) {
                rr[l] = sb[l * TW + col];
                if (KIND == 1 && !fresh) pp[l] = sb[F_P + l * TW + col];
                if (KIND == 2 || !fresh) vq[l] = sb[F_V + l * TW + col];
                const double2 ud = *reinterpret_cast<const double2*>(sb + F_UD + l * 2 * TW + 2 * col);
                uu[l] = ud.x;
                dd[l] = ud.y;
            }
            fence_proxy_async_smem();
            mbar_arrive(&emptyF[cslot]);
            if (++cslot == NSF) { cslot = 0; cphase ^= 1u; }
            V cb[KS], yb[KS], fb[KS];
#pragma unroll
            for (int e = 0; e < KS; ++e) {
                const int k = k0 + e;
                V f;
                if (KIND == 1) f = fresh ? rr[e] : fma(beta, fma(-omega, vq[e], pp[e]), rr[e]);
                else f = fma(-alpha, vq[e], rr[e]);
                V cc, y;
                if (k == 0) {
                    cc = uu[e];
                    y = f;
                } else {
                    const V inv = rcp_fast<V>(fma(-dd[e], cprev, 1.0));
                    cc = uu[e] * inv;
                    y = fma(-dd[e], yprev, f) * inv;
                }
                if (k >= nz) cc = y = 0.0;  // padded levels: z = 0 above the top
                cb[e] = cc; yb[e] = y; fb[e] = f;
                cprev = cc;
                yprev = y;
            }
            V* pk = pw + (int64_t)k0 * nx;
            if (uni && k0 + KS <= nz) {
#pragma unroll
                for (int e = 0; e < KS; ++e) __stcg(pk + e * nx, fb[e]);
            } else {
#pragma unroll
                for (int e = 0; e < KS; ++e)
                    if (act && k0 + e < nz) __stcg(pk + e * nx, fb[e]);
            }
            tm_st8d(tl + (uint32_t)(2 * k0), cb);
            if (sync_step >= 0) {  // the S warps read s (TMEM slot us) and z(r_{m-1}) of this chunk
                mbar_wait(&sread[c], (uint32_t)(sync_step & 1));
                MA_TFENCE_AFTER();
            }
#pragma unroll
            for (int e = 0; e < KS; ++e) zr[(k0 + e) * M6_RING_W] = yb[e];
            if (KIND == 2) tm_st8d(tS(us) + (uint32_t)(2 * k0), fb);
        };
        auto back_row = [&](V* zr, V* zw, int x) {
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            V zn = 0.0;
            for (int k0 = NZ4 - KS; k0 >= 0; k0 -= KS) {
                float cw[8];
                V yb[KS];
                tm_ld8_nw(tl + (uint32_t)(2 * k0), cw);
#pragma unroll
                for (int e = 0; e < KS; ++e) yb[e] = zr[(k0 + e) * M6_RING_W];
                tm_wait_ld();
#pragma unroll
                for (int e = KS - 1; e >= 0; --e) {
                    const int k = k0 + e;
                    zn = (k == nz - 1) ? yb[e] : fma(-join_d(cw[2 * e], cw[2 * e + 1]), zn, yb[e]);
                    if (k >= nz) zn = 0.0;
                    yb[e] = zn;
                }
#pragma unroll
                for (int e = 0; e < KS; ++e) zr[(k0 + e) * M6_RING_W] = yb[e];
                V* zk = zw + (int64_t)k0 * nx;
                if (uni && k0 + KS <= nz) {
#pragma unroll
                    for (int e = 0; e < KS; ++e) __stcg(zk + e * nx, yb[e]);
                } else {
#pragma unroll
                    for (int e = 0; e < KS; ++e)
                        if (act && k0 + e < nz) __stcg(zk + e * nx, yb[e]);
                }
            }
            MA_TFENCE_BEFORE();
            mbar_arrive(&zready[x & 1]);
            if (x >= 2) mbar_wait(&pubd[x & 1], (uint32_t)(((x - 2) >> 1) & 1));
            mbar_arrive(&zdone[x & 1]);
        };
        auto T_row = [&](int x, int sync_step) {
            const int jr = row_of(x);
            V* zr = slot_ptr(x) + 1 + col;
            V* pw = Pw + (int64_t)jr * g.row + i;
            cprev = yprev = 0.0;
            for (int c = 0; c < nch; ++c) fwd_chunk(c * KS, c, zr, pw, x & 1, sync_step);
            back_row(zr, Zw + (int64_t)jr * g.row + i, x);
        };
        T_row(0, -1);
        if (L >= 2) T_row(1, -1);
        for (int m = 0; m + 2 < L; ++m) T_row(m + 2, m);
    } else {
        // ============================ stencil warps ============================
        constexpr int NQ = KIND == 1 ? 1 : 3;
        V* __restrict__ Yw = KIND == 1 ? vv.v : vv.t;
        const int T128 = g.tiles;  // 128-column slot tiles: this CTA fills half (t & 1) of slot t / 2
        const int64_t per_q = (int64_t)nyl * T128 * 4;
        int cslot = 0;
        uint32_t cphase = 0;
        auto wait_flag = [&](int row, int tile) {
            const int* f = flags + (int64_t)row * T + tile;
            while (ld_acquire(f) != epoch) __nanosleep(40);
        };
        auto load_row = [&](V* dst, int row) {
            const V* src = Zw + (int64_t)row * g.row + i;
            for (int k = 0; k < nz; ++k) dst[k * M6_RING_W] = __ldcg(src + (int64_t)k * nx);
        };
        // E / W halo of r_x from hbuf into its ring slot, then free hbuf[x & 1]
        auto copy_halo = [&](int x) {
            mbar_wait(&hready[x & 1], (uint32_t)((x >> 1) & 1));
            V* zr = slot_ptr(x);
            for (int k = tid; k < nz; k += M6_CONS) {
                zr[k * M6_RING_W] = hbuf[x & 1][0][k];
                zr[k * M6_RING_W + w + 1] = hbuf[x & 1][1][k];
            }
            mbar_arrive(&hfree[x & 1]);
        };
        for (int m = 0; m < L; ++m) {
            const int j = row_of(m);
            const int64_t jg = g.j0 + j;
            const bool hasN = jg < g.ny - 1, hasS = jg > 0;
            if (m == 0) mbar_wait(&zready[0], 0u);
            if (m + 1 < L) mbar_wait(&zready[(m + 1) & 1], (uint32_t)(((m + 1) >> 1) & 1));
            MA_TFENCE_AFTER();
            V* zC0 = slot_ptr(m);
            V* zN0 = hasN ? (dir > 0 ? slot_ptr(m + 1) : slot_ptr(m - 1)) : zC0;
            V* zS0 = hasS ? (dir > 0 ? slot_ptr(m - 1) : slot_ptr(m + 1)) : zC0;
            const bool ld_prev = m == 0 && (dir > 0 ? hasS : hasN);
            const bool ld_next = m == L - 1 && (dir > 0 ? hasN : hasS);
            if (m == 0 || ld_next) {
                if (tid == 0) {
                    if (ld_prev && j - dir >= 0 && j - dir < nyl) wait_flag(j - dir, t);
                    if (ld_next && j + dir >= 0 && j + dir < nyl) wait_flag(j + dir, t);
                }
                cons6_bar();
                if (m == 0) copy_halo(0);
                if (ld_prev) load_row(slot_ptr(m - 1) + 1 + col, j - dir);
                if (ld_next) load_row(slot_ptr(m + 1) + 1 + col, j + dir);
                cons6_bar();
            }
            const V* zC = zC0 + 1 + col;
            const V* zN = zN0 + 1 + col;
            const V* zS = zS0 + 1 + col;
            V* yw = Yw + (int64_t)j * g.row + i;
            const int us = m & 1;
            double acc[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
            V zprev = 0.0;
            for (int c = 0; c < nch; ++c) {
                const int k0 = c * KS;
                float sw[8];
                if (KIND == 2) tm_ld8_nw(tS(us) + (uint32_t)(2 * k0), sw);
                mbar_wait(&fullS[cslot], cphase);
                const V* sbS = stS + (size_t)cslot * SSD;
                V bE[KS], bW[KS], bN[KS], bS[KS], bU[KS], bD[KS], ax[KS];
                V zc[KS + 1], zE[KS], zWv[KS], zNv[KS], zSv[KS], av[KS];
#pragma unroll
                for (int l = 0; l < KS; ++l) {
                    const double2 ew = *reinterpret_cast<const double2*>(sbS + l * 4 * TW + 4 * col);
                    const double2 ns = *reinterpret_cast<const double2*>(sbS + l * 4 * TW + 4 * col + 2);
                    const double2 ud = *reinterpret_cast<const double2*>(sbS + S_UD + l * 2 * TW + 2 * col);
                    bE[l] = ew.x; bW[l] = ew.y; bN[l] = ns.x; bS[l] = ns.y; bU[l] = ud.x; bD[l] = ud.y;
                    if (KIND == 1) ax[l] = sbS[S_RH + l * TW + col];
                }
#pragma unroll
                for (int e = 0; e < KS; ++e) {
                    const int ko = (k0 + e) * M6_RING_W;
                    zc[e] = zC[ko];
                    zE[e] = zC[ko + 1];
                    zWv[e] = zC[ko - 1];
                    zNv[e] = zN[ko];
                    zSv[e] = zS[ko];
                }
                zc[KS] = zC[min(k0 + KS, nz - 1) * M6_RING_W];
                if (KIND == 2) tm_wait_ld();
                MA_TFENCE_BEFORE();
                fence_proxy_async_smem();
                mbar_arrive(&emptyS[cslot]);
                if (++cslot == NSS) { cslot = 0; cphase ^= 1u; }
                mbar_arrive(&sread[c]);  // the F warps may now overwrite this chunk
                if (KIND == 2) {
#pragma unroll
                    for (int e = 0; e < KS; ++e) ax[e] = join_d(sw[2 * e], sw[2 * e + 1]);
                }
#pragma unroll
                for (int e = 0; e < KS; ++e) {
                    const int k = k0 + e;
                    const V zp = (k + 1 < nz) ? zc[e + 1] : zc[e];  // multiplied by U = 0 on the top level
                    V a = zc[e];
                    a = fma(bE[e], zE[e], a);
                    a = fma(bW[e], zWv[e], a);
                    a = fma(bN[e], zNv[e], a);
                    a = fma(bS[e], zSv[e], a);
                    a = fma(bU[e], zp, a);
                    a = fma(bD[e], zprev, a);  // zprev = 0 at k = 0 (D = 0 there)
                    zprev = zc[e];
                    av[e] = a;
                    if (act && k < nz) {
                        if (KIND == 1) {
                            acc_dot<0>(acc[0], ax[e], a);
                        } else {
                            acc_dot<0>(acc[0], a, ax[e]);
                            acc_dot<0>(acc[1], a, a);
                            acc_dot<0>(acc[2], ax[e], ax[e]);
                        }
                    }
                }
                V* yk = yw + (int64_t)k0 * nx;
                if (uni && k0 + KS <= nz) {
#pragma unroll
                    for (int e = 0; e < KS; ++e) __stcg(yk + e * nx, av[e]);
                } else {
#pragma unroll
                    for (int e = 0; e < KS; ++e)
                        if (act && k0 + e < nz) __stcg(yk + e * nx, av[e]);
                }
            }
            // warp sums (k_stencil's shuffle tree) into the half-slots: warp (t & 1) * 2 + warp of the
            // 128-column slot t / 2; the finaliser adds the four in k_stencil's order
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                double a = acc[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
                if (lane == 0) hslots[q * per_q + ((int64_t)j * T128 + (t >> 1)) * 4 + (t & 1) * 2 + warp] = a;
            }
            if (m + 1 < L) copy_halo(m + 1);
            cons6_bar();  // ring halo columns are rewritten by the next step
        }
    }
    // ---- all compute warps: release TMEM ----
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    asm volatile("bar.sync 2, 128;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
    }
}

}  // namespace eg
