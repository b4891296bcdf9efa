// sipg_apply2.cuh — K1/K4/K6 v3: the hot kernel, matrix-free sum-factorised SIPG operator
// apply (vector viscous operator, PAPER.md:1055-1111 eqn:viscous_term_weak; scalar Poisson,
// PAPER.md:713-758 eqn:pressure_step_weak) with fused epilogues (plain apply, residual
// b - A x, Chebyshev-Jacobi update of SURVEY §8(c) c1.6).
//
// Same cell-centric algorithm as v2 (team of n^2 threads per cell, thread (a,b) owns the
// z-column x=a, y=b in registers, faces evaluated from the cell's own side, no atomics), with
// the shared-memory traffic redesigned after the v2 ncu source profile (L1
// wavefronts 80 % of peak, 4-way bank conflicts on the face accumulator, per-thread
// uncoalesced neighbour x-lines as the top stall):
//  * every volume array is kept twice, [c][z][y][x] and transposed [c][z][x][y], with rows
//    padded to an even length RS and planes to PS (PS/2 odd): every contraction reads whole
//    rows with 16-byte loads (broadcast across the team), and rows read by 16 different lanes
//    are bank-conflict free;
//  * x- and y-face contributions are written once per direction (no read-modify-write, no
//    zeroing) into a row-major buffer and folded into the column registers by the owners;
//  * a neighbour that sits in the same CTA (consecutive cells: the x-neighbours of structured
//    meshes) is read from shared memory; other neighbour x-lines are read as 16-byte rows;
//  * faces one at a time (traces + tangential coefficients of one face in shared memory), the
//    general-geometry flux computed neighbour side first so J^-1 of both sides is never live
//    together with both physical gradients.
#pragma once
#include "common.cuh"

#ifndef DGVV_FACE_TMA
#define DGVV_FACE_TMA 1   // stage the general-geometry face metric with TMA bulk copies
#endif
#ifndef DGVV_FACE_TMA_CART
#define DGVV_FACE_TMA_CART 1   // stage the Cartesian face viscosities with TMA bulk copies
#endif
#ifndef USE_ST
#define USE_ST 0          // keep a transposed [c][z][x][y] copy of the cell (16-byte y-lines)
#endif
#ifndef DGVV_NBCART_EARLY
#define DGVV_NBCART_EARLY 1   // Cartesian: the two neighbours' geometry of a direction loaded at its start
#endif
#ifndef DGVV_NU_EARLY
#define DGVV_NU_EARLY 1       // Cartesian: load the column's cell-point coefficients with the column
#endif
#ifndef DGVV_CARTF
#define DGVV_CARTF 1          // Cartesian: neighbour 1/h_d and max(H, H_nb) from the cell's own record
#endif
#ifndef DGVV_NB_L2PF
#define DGVV_NB_L2PF 1        // L2 prefetch (per-thread lines) of neighbours more than one resident wave ahead
#endif
#ifndef DGVV_NUF_EARLY
#define DGVV_NUF_EARLY 1      // Cartesian without the TMA stage: a direction's face coefficients loaded at its start
#endif
#ifndef DGVV_ZTR
#define DGVV_ZTR 1            // Cartesian divergence form: z-face own tangential derivatives from the volume term
#endif
#ifndef DGVV_QUAD_SWIZZLE
#define DGVV_QUAD_SWIZZLE 1   // n = 4: lane quads cover 2 x 2 blocks of columns (see the kernel)
#endif


namespace dgvv {

template <int n>
struct Lay {
  static constexpr int n2 = n * n, n3 = n * n * n;
  static constexpr int RS = (n + 1) & ~1;                          // row stride (even)
  static constexpr int PS0 = n * RS;
  static constexpr int PS = ((PS0 / 2) % 2 == 1) ? PS0 : PS0 + 2;  // plane stride, PS/2 odd
  static constexpr int CST = n * PS;                               // component stride
  static constexpr int FA = n * RS;                                // one face array [n][RS]
};

template <int n, int NC, int FORM, int GEO>
struct Apply2Cfg {
  using L = Lay<n>;
  static constexpr int NT = (GEO == 1) ? NC : (FORM == 0 ? 1 : 0);
  static constexpr int VOL = NC * L::CST;
  static constexpr int FB = 8 * NT * L::FA;                        // [2 faces][Tm Tp G1 G2T]
  static constexpr int RW = (2 * VOL > VOL + FB) ? 2 * VOL : VOL + FB;
  // general geometry, n even: the face metric of one direction (own J^-1 and nu*dA of both
  // faces, the two neighbours' of their opposite faces) is staged by TMA bulk copies
  static constexpr bool TMA = (GEO == 1) && (n % 2 == 0) && (DGVV_FACE_TMA != 0);
  // Cartesian divergence form, n even: the face viscosities of all six faces (own, and each
  // neighbour's opposite face) are staged by TMA bulk copies issued at kernel start
  // (DGVV_FACE_TMA_CART; measured: C5 3246 -> 3040 us; slower for the scalar Poisson operator and
  // as per-direction stages)
  static constexpr bool TMAC = (GEO == 0) && (n % 2 == 0) && (FORM == 0) && (DGVV_FACE_TMA_CART != 0);
  static constexpr bool STAGE = TMA || TMAC;
  static constexpr int STG = TMA ? 40 * L::n2 : (TMAC ? 12 * L::n2 : 0);
  static constexpr int CS = (1 + USE_ST) * VOL + RW + STG;         // doubles of smem per cell
};

// --- TMA (cp.async.bulk) + mbarrier helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
  asm volatile("{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
               " @!P bra WAIT_%=;\n}" ::"r"(smem_u32(m)), "r"(parity) : "memory");
}

// 2-element vector type of the real type (16-byte rows for double, 8-byte for float)
template <typename R> struct V2;
template <> struct V2<double> {
  using t = double2;
  static __device__ __forceinline__ t mk(double a, double b) { return make_double2(a, b); }
};
template <> struct V2<float> {
  using t = float2;
  static __device__ __forceinline__ t mk(float a, float b) { return make_float2(a, b); }
};

// row of n values (2-element aligned) into registers
template <int n, typename R>
__device__ __forceinline__ void ld_row(const R* __restrict__ r, R (&x)[n]) {
#pragma unroll
  for (int k = 0; k + 1 < n; k += 2) {
    const typename V2<R>::t v = *reinterpret_cast<const typename V2<R>::t*>(r + k);
    x[k] = v.x;
    x[k + 1] = v.y;
  }
  if constexpr (n & 1) x[n - 1] = r[n - 1];
}
template <int n, typename R>
__device__ __forceinline__ void ldg_row(const R* __restrict__ r, R (&x)[n]) {
  if constexpr (sizeof(R) == 8 && n % 4 == 0) {
    // 256-bit loads (sm_100: LDG.E.ENL2.256): one instruction and one pass over each 32-byte
    // sector per 4 doubles (two 128-bit loads touched every sector twice); rows are 32-B aligned
    // (vectors 32-B aligned, checked by the ABI)
#pragma unroll
    for (int k = 0; k < n; k += 4)
      asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
          : "=d"(x[k]), "=d"(x[k + 1]), "=d"(x[k + 2]), "=d"(x[k + 3]) : "l"(r + k));
    return;
  } else if constexpr (sizeof(R) == 4 && n % 4 == 0) {
#pragma unroll
    for (int k = 0; k < n; k += 4) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(r + k));
      x[k] = v.x; x[k + 1] = v.y; x[k + 2] = v.z; x[k + 3] = v.w;
    }
    return;
  }
#pragma unroll
  for (int k = 0; k + 1 < n; k += 2) {
    const typename V2<R>::t v = __ldg(reinterpret_cast<const typename V2<R>::t*>(r + k));
    x[k] = v.x;
    x[k + 1] = v.y;
  }
  if constexpr (n & 1) x[n - 1] = __ldg(r + n - 1);
}
template <int n, typename R>
__device__ __forceinline__ void st_row(R* __restrict__ r, const R (&x)[n]) {
#pragma unroll
  for (int k = 0; k + 1 < n; k += 2) *reinterpret_cast<typename V2<R>::t*>(r + k) = V2<R>::mk(x[k], x[k + 1]);
  if constexpr (n & 1) r[n - 1] = x[n - 1];
}
template <int n, typename R>
__device__ __forceinline__ R rowdot(const R* __restrict__ r, const R (&w)[n]) {
  R x[n];
  ld_row<n>(r, x);
  R s = R(0);
#pragma unroll
  for (int k = 0; k < n; ++k) s = fma(w[k], x[k], s);
  return s;
}

template <typename R, int n, int NC, int FORM, int GEO, int CPB, int MINB, bool MASS, bool CONV = false, bool GTR = false>
__global__ void __launch_bounds__(CPB * n * n, MINB)
sipg_apply2_kernel(const ApplyArgsT<R> A) {
  static_assert(FORM == 1 || NC == 3, "divergence form needs 3 components");
  static_assert(!CONV || NC == 3, "the convective term acts on the velocity");
  using L = Lay<n>;
  using Cf = Apply2Cfg<n, NC, FORM, GEO>;
  constexpr int n2 = L::n2, n3 = L::n3, RS = L::RS, PS = L::PS, CST = L::CST, FA = L::FA;
  constexpr int NT = Cf::NT, VOL = Cf::VOL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* smem = reinterpret_cast<R*>(smem_raw);
  __shared__ __align__(16) R sD[n * RS];    // sD[i][k]  = l_k'(x_i)
  __shared__ __align__(16) R sDT[n * RS];   // sDT[i][k] = l_i'(x_k)
  __shared__ int sid[CPB];
  const Tab1D& T = c_tab[n];

  const int lc = threadIdx.x / n2;
  const int pr = threadIdx.x - lc * n2;
  // Lane -> column (a, b).  Shared-memory cost on B200 (measured, scripts/lds_patterns.cu, DESIGN.md
  // §6): a 64-bit load costs one wavefront per 128 B of distinct data summed over the warp's lane
  // quads (4 consecutive lanes share one read port), a 128-bit load at least two.  With a fastest
  // (p = a + n b) a quad shares its row (x-direction loads: 1 wavefront) but reads 4 different
  // columns (y-direction loads: 2).  For n = 4 the quad covers a 2 x 2 block of (a, b) instead:
  // 2 distinct rows and 2 distinct columns per quad, one wavefront per 64-bit load either way.
  // n = 6 likewise: quad q = pr / 4 (9 per team; a team of 36 starts on a quad boundary) covers the
  // 2 x 2 block (2 (q % 3), 2 (q / 3)).  n = 5 teams (25 lanes) straddle quads: natural order.
  constexpr bool SWZ = DGVV_QUAD_SWIZZLE && (n == 4 || n == 6);
  const int a = !SWZ ? pr % n : (n == 4 ? ((pr & 1) | ((pr >> 1) & 2)) : 2 * ((pr >> 2) % 3) + (pr & 1));
  const int b = !SWZ ? pr / n : (n == 4 ? (((pr >> 1) & 1) | ((pr >> 2) & 2)) : 2 * ((pr >> 2) / 3) + ((pr >> 1) & 1));
  const int p = a + n * b;                          // the column's point index in the cell block
  const int slot_raw = blockIdx.x * CPB + lc;
  const bool active = slot_raw < A.n_proc;
  const int slot = active ? slot_raw : (A.n_proc - 1);
  const int cell = A.cell_list ? A.cell_list[slot] : A.cell_base + slot;

  for (int i = threadIdx.x; i < n * RS; i += blockDim.x) {
    const int r = i / RS, k = i - r * RS;
    sD[i] = k < n ? R(T.D[r * DGVV_NMAX + k]) : R(0.0);
    sDT[i] = k < n ? R(T.D[k * DGVV_NMAX + r]) : R(0.0);
  }
  if (p == 0) sid[lc] = active ? cell : -1;
  __shared__ __align__(8) uint64_t mbar[CPB];
  R* stg = smem + lc * Cf::CS + (Cf::CS - Cf::STG);   // face-metric stage (TMA)
  // issue the TMA bulk copies of direction d's face metric for this cell (thread p == 0)
  auto stage_issue = [&](int d, const int (&nb)[6]) {
    if constexpr (Cf::TMAC) {          // all six faces at once (issued at kernel start, d ignored)
      constexpr uint32_t BN = n2 * sizeof(R);
      uint32_t bytes = 6 * BN;
#pragma unroll
      for (int f = 0; f < 6; ++f) bytes += nb[f] >= 0 ? BN : 0;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&mbar[lc], bytes);
      tma_load_1d(stg, A.nu_face + (size_t)cell * 6 * n2, 6 * BN, &mbar[lc]);
#pragma unroll
      for (int f = 0; f < 6; ++f)
        if (nb[f] >= 0) tma_load_1d(stg + (6 + f) * n2, A.nu_face + ((size_t)nb[f] * 6 + (f ^ 1)) * n2, BN, &mbar[lc]);
    }
    if constexpr (Cf::TMA) {
      constexpr uint32_t BJ = 9 * n2 * sizeof(R), BN = n2 * sizeof(R);
      uint32_t bytes = 2 * (BJ + BN);
#pragma unroll
      for (int s = 0; s < 2; ++s) bytes += nb[2 * d + s] >= 0 ? BJ + BN : 0;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&mbar[lc], bytes);
      tma_load_1d(stg, A.fJi + ((size_t)cell * 6 + 2 * d) * 9 * n2, 2 * BJ, &mbar[lc]);
      tma_load_1d(stg + 18 * n2, A.nu_face + ((size_t)cell * 6 + 2 * d) * n2, 2 * BN, &mbar[lc]);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int nb_ = nb[2 * d + s];
        if (nb_ >= 0) {
          const int fo = (2 * d + s) ^ 1;
          tma_load_1d(stg + 20 * n2 + s * 9 * n2, A.fJi + ((size_t)nb_ * 6 + fo) * 9 * n2, BJ, &mbar[lc]);
          tma_load_1d(stg + 38 * n2 + s * n2, A.nu_face + ((size_t)nb_ * 6 + fo) * n2, BN, &mbar[lc]);
        }
      }
    }
  };

  R* su = smem + lc * Cf::CS;      // values     [NC][z][y][x]
  R* sT = su + VOL;                // transposed [NC][z][x][y] (USE_ST)
  R* WK = su + (1 + USE_ST) * VOL;  // work: W1 | W2T (volume); Y | face buffers (faces)

  R ucol[NC][n], y[NC][n];
  {
    const R* gsrc = A.src + (size_t)cell * NC * n3;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z) {
        const R v = __ldg(gsrc + c * n3 + z * n2 + p);
        ucol[c][z] = v;
        y[c][z] = R(0.0);
        su[c * CST + z * PS + b * RS + a] = v;
        if (USE_ST) sT[c * CST + z * PS + a * RS + b] = v;
      }
  }
  // the cell-point coefficient of the column, loaded with the column (its latency overlaps the
  // column loads instead of stalling the volume term)
  R nuq[(GEO == 0 && DGVV_NU_EARLY) ? n : 1];
  if constexpr (GEO == 0 && DGVV_NU_EARLY) {
#pragma unroll
    for (int z = 0; z < n; ++z) nuq[z] = A.nu_cell[(size_t)cell * n3 + z * n2 + p];
  }
  R ih[3] = {0, 0, 0}, vol = R(0.0), Hm;
  if constexpr (GEO == 0) {
    const R* cg = A.cart + (size_t)cell * CART_STRIDE;
    ih[0] = cg[0]; ih[1] = cg[1]; ih[2] = cg[2]; Hm = cg[3]; vol = cg[4];
  } else {
    Hm = A.Hcell[cell];
  }
  int nbf[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) nbf[f] = __ldg(A.nbr + cell * 6 + f);
  if constexpr (DGVV_NB_L2PF != 0 && n != 4) {
    // L2 prefetch of the neighbour blocks more than one resident wave (148 SMs x MINB CTAs x CPB
    // cells) ahead in the cell order: no resident CTA has requested them yet, so their face lines
    // would come from HBM (+z on C3's 64^3 cube, 4096 cells ahead: C3 -1.3 %).  Nearer ones are
    // being loaded by their own CTA; prefetching those measured slower (C5 +x, 2048 ahead: +0.7 %).
    // One 128-B line per thread.  Not built for n = 4: the code alone costs C5 1.2 % (registers).
    constexpr int BLK = NC * n3 * (int)sizeof(R), NL = (BLK + 127) / 128, WAVE = 148 * MINB * CPB;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int nbv = nbf[f];
      if (nbv > cell + WAVE && nbv < A.n_owned) {
        const char* base = reinterpret_cast<const char*>(A.src + (size_t)nbv * NC * n3);
        for (int l = p; l < NL; l += n2) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + 128 * l));
      }
    }
  }
  if constexpr (Cf::STAGE) {
    if (p == 0) {
      mbar_init(&mbar[lc], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      stage_issue(2, nbf);      // z faces first: latency hidden by the volume term (issuing it inside
                                // the volume term instead measured +1-4 %)
    }
  }
  __syncthreads();

  // Cartesian divergence form: the tangential derivatives of the own trace of u_z on the two
  // z faces are the z-traces of the reference x- and y-derivatives of u_z the volume term computes
  // along this thread's own column (linearity of the trace): accumulated there, they replace the
  // z-faces' own trace round trip through shared memory (store + row and column contractions).
  // Measured C5 2605 -> 2589 us
  constexpr bool ZTR = (GEO == 0) && (FORM == 0) && (n % 2 == 0) && (DGVV_ZTR != 0);   // n = 5: +0.5 % (C3), not built
  R ztr[2][2] = {{R(0.0), R(0.0)}, {R(0.0), R(0.0)}};   // [face s][x / y derivative]
  // =============================================================== volume term
  {
    R Da[n], Db[n];
    ld_row<n>(sD + a * RS, Da);
    ld_row<n>(sD + b * RS, Db);
    const R wab = R(T.w[a]) * R(T.w[b]);
#pragma unroll
    for (int z = 0; z < n; ++z) {
      const int q = z * n2 + p;
      R gxi[NC][3];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        gxi[c][0] = rowdot<n>(su + c * CST + z * PS + b * RS, Da);
        if (USE_ST) {
          gxi[c][1] = rowdot<n>(sT + c * CST + z * PS + a * RS, Db);
        } else {
          R sy = R(0.0);
#pragma unroll
          for (int k = 0; k < n; ++k) sy = fma(Db[k], su[c * CST + z * PS + k * RS + a], sy);
          gxi[c][1] = sy;
        }
        R sz = R(0.0);
#pragma unroll
        for (int k = 0; k < n; ++k) sz = fma(R(T.D[z * DGVV_NMAX + k]), ucol[c][k], sz);
        gxi[c][2] = sz;
      }
      if constexpr (ZTR) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          ztr[0][j] = fma(R(T.l0[z]), gxi[2][j], ztr[0][j]);
          ztr[1][j] = fma(R(T.l1[z]), gxi[2][j], ztr[1][j]);
        }
      }
      R Ji[9], w;
      if constexpr (GEO == 0) {
        if constexpr (DGVV_NU_EARLY) w = nuq[z] * wab * R(T.w[z]) * vol;
        else w = A.nu_cell[(size_t)cell * n3 + q] * wab * R(T.w[z]) * vol;
      } else {
        const R* vm = A.vJi + (size_t)cell * 9 * n3 + q;
#pragma unroll
        for (int r = 0; r < 9; ++r) Ji[r] = __ldg(vm + r * n3);
        w = A.nu_cell[(size_t)cell * n3 + q];         // nu * JxW
      }
      if constexpr (CONV) {
        // f4 (fused): + alpha_c JxW (w.grad) u at the point (collocation: the test function is the
        // point value), from the stored reference transport direction wref = JxW J^-1 w
        const R* gw = A.wref + (size_t)cell * 3 * n3 + q;
        const R ac = R(A.alpha_c);
        const R wr0 = ac * __ldg(gw), wr1 = ac * __ldg(gw + n3), wr2 = ac * __ldg(gw + 2 * n3);
#pragma unroll
        for (int c = 0; c < NC; ++c) y[c][z] = fma(gxi[c][0], wr0, fma(gxi[c][1], wr1, fma(gxi[c][2], wr2, y[c][z])));
      }
      R G[NC][3];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          if constexpr (GEO == 0) G[c][j] = gxi[c][j] * ih[j];
          else G[c][j] = gxi[c][0] * Ji[j] + gxi[c][1] * Ji[3 + j] + gxi[c][2] * Ji[6 + j];
        }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        R Tc[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          if constexpr (FORM == 0) Tc[j] = w * (G[c][j] + G[j][c]);
          else Tc[j] = w * G[c][j];
        }
        R F[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          if constexpr (GEO == 0) F[k] = Tc[k] * ih[k];
          else F[k] = Tc[0] * Ji[3 * k] + Tc[1] * Ji[3 * k + 1] + Tc[2] * Ji[3 * k + 2];
        }
        WK[c * CST + z * PS + b * RS + a] = F[0];               // W1  [c][z][y][x]
        WK[VOL + c * CST + z * PS + a * RS + b] = F[1];         // W2T [c][z][x][y]
#pragma unroll
        for (int z2 = 0; z2 < n; ++z2) y[c][z2] = fma(R(T.D[z * DGVV_NMAX + z2]), F[2], y[c][z2]);
      }
    }
    __syncthreads();
    R DTa[n], DTb[n];
    ld_row<n>(sDT + a * RS, DTa);
    ld_row<n>(sDT + b * RS, DTb);
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int z = 0; z < n; ++z)
        y[c][z] += rowdot<n>(WK + c * CST + z * PS + b * RS, DTa) + rowdot<n>(WK + VOL + c * CST + z * PS + a * RS, DTb);
    __syncthreads();
  }

  // =============================================================== face terms
  // Faces in opposite pairs (-d,+d): one pass over each normal line gives the own traces of
  // both faces; the traces of both faces go to smem together (one barrier), then the
  // tangential coefficients of both (second barrier).  Order z, x, y: the z pair works on the
  // column registers (ucol dies after it).  buffers: [s][Tm | Tp | G1 | G2T][NT][FA]
#pragma unroll
  for (int dd = 0; dd < 3; ++dd) {
    const int d = (dd == 0) ? 2 : dd - 1;
    const int t1 = face_t1(d), t2 = face_t2(d);
    R ihq[2][3], Hq[2];                 // DGVV_NBCART_EARLY: neighbours' 1/h and H, loaded up front
    if constexpr (GEO == 0 && DGVV_NBCART_EARLY) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if constexpr (DGVV_CARTF) {
          // from this cell's own record: the neighbour's 1/h_d and max(H, H_nb) (a conforming
          // neighbour shares the tangential extents)
          const R* cf = A.cart + (size_t)cell * CART_STRIDE + CART_FACE + 2 * (2 * d + s);
          ihq[s][0] = ih[0]; ihq[s][1] = ih[1]; ihq[s][2] = ih[2];
          ihq[s][d] = cf[0]; Hq[s] = cf[1];
        } else {
          const int nbv = nbf[2 * d + s];
          const R* cg = A.cart + (size_t)(nbv >= 0 ? nbv : cell) * CART_STRIDE;
          ihq[s][0] = cg[0]; ihq[s][1] = cg[1]; ihq[s][2] = cg[2]; Hq[s] = cg[3];
        }
      }
    }
    // Cartesian without the TMA stage (n odd, Laplace form): this direction's face coefficients
    // (own and the neighbour's at each face point) loaded at its start, so their latency overlaps
    // the trace phase (ncu C3: 13 % of the stall samples waited on them in the flux)
    constexpr bool NUF_EARLY = (GEO == 0) && !Cf::TMAC && (DGVV_NUF_EARLY != 0);
    R nuf_m[2], nuf_p[2];
    if constexpr (NUF_EARLY) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int f = 2 * d + s, nbv = nbf[f];
        nuf_m[s] = A.nu_face[((size_t)cell * 6 + f) * n2 + p];
        nuf_p[s] = nbv >= 0 ? A.nu_face[((size_t)nbv * 6 + (f ^ 1)) * n2 + p] : nuf_m[s];
      }
    }

    R um[2][NC], dm[2][NC], up[2][NC], dp[2][NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      R x[n];
      if (d == 2) {
#pragma unroll
        for (int i = 0; i < n; ++i) x[i] = ucol[c][i];
      } else if (d == 0 || USE_ST) {
        ld_row<n>((d == 0 ? su : sT) + c * CST + b * PS + a * RS, x);
      } else {
#pragma unroll
        for (int i = 0; i < n; ++i) x[i] = su[c * CST + b * PS + i * RS + a];
      }
      R v0 = R(0.0), g0 = R(0.0), v1 = R(0.0), g1 = R(0.0);
#pragma unroll
      for (int i = 0; i < n; ++i) {
        v0 = fma(R(T.l0[i]), x[i], v0); g0 = fma(R(T.d0[i]), x[i], g0);
        v1 = fma(R(T.l1[i]), x[i], v1); g1 = fma(R(T.d1[i]), x[i], g1);
      }
      um[0][c] = v0; dm[0][c] = g0; um[1][c] = v1; dm[1][c] = g1;
    }
    // neighbour traces: from the neighbour's smem copy when it sits in this CTA, else global
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int nbv = nbf[2 * d + s];
      if (nbv >= 0) {
        const double* lO = s ? T.l0 : T.l1;
        const double* dO = s ? T.d0 : T.d1;
        const int sl = lc + (nbv - cell);
        const bool in_cta = sl >= 0 && sl < CPB && sid[sl] == nbv;
        const R* pn = nbv < A.n_owned ? A.src + (size_t)nbv * NC * n3
                                           : A.ghost + (size_t)(nbv - A.n_owned) * NC * n3;
        const R* ns = smem + (in_cta ? sl : 0) * Cf::CS;
        if (GTR && nbv >= A.n_owned) {            // exchanged face traces of the ghost neighbour (boundary launch)
          const R* tr = A.gtr + (size_t)A.gslot[(nbv - A.n_owned) * 6 + ((2 * d + s) ^ 1)] * NC * 2 * n2 + p;
#pragma unroll
          for (int c = 0; c < NC; ++c) { up[s][c] = tr[2 * c * n2]; dp[s][c] = tr[(2 * c + 1) * n2]; }
          continue;
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          R x[n];
          if (in_cta) {
            if (d == 2) {
#pragma unroll
              for (int i = 0; i < n; ++i) x[i] = ns[c * CST + i * PS + b * RS + a];
            } else if (d == 0 || USE_ST) {
              ld_row<n>(ns + (d == 0 ? 0 : VOL) + c * CST + b * PS + a * RS, x);
            } else {
#pragma unroll
              for (int i = 0; i < n; ++i) x[i] = ns[c * CST + b * PS + i * RS + a];
            }
          } else {
            if (d == 0) {
              if constexpr ((n & 1) == 0) ldg_row<n>(pn + c * n3 + b * n2 + a * n, x);
              else {
#pragma unroll
                for (int i = 0; i < n; ++i) x[i] = __ldg(pn + c * n3 + b * n2 + a * n + i);
              }
            } else if (d == 1) {
#pragma unroll
              for (int i = 0; i < n; ++i) x[i] = __ldg(pn + c * n3 + b * n2 + i * n + a);
            } else {
#pragma unroll
              for (int i = 0; i < n; ++i) x[i] = __ldg(pn + c * n3 + i * n2 + p);
            }
          }
          R v = R(0.0), g = R(0.0);
#pragma unroll
          for (int i = 0; i < n; ++i) { v = fma(R(lO[i]), x[i], v); g = fma(R(dO[i]), x[i], g); }
          up[s][c] = v; dp[s][c] = g;
        }
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) { up[s][c] = -um[s][c]; dp[s][c] = dm[s][c]; }
      }
    }
    if constexpr (NT > 0) {
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int c = (GEO == 1) ? t : d;
          if (!(ZTR && d == 2)) WK[VOL + ((s * 4 + 0) * NT + t) * FA + b * RS + a] = um[s][c];
          WK[VOL + ((s * 4 + 1) * NT + t) * FA + b * RS + a] = up[s][c];
        }
      __syncthreads();
    }

    R fv[2][NC], gn[2][NC];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int f = 2 * d + s;
      const int nbv = nbf[f];
      const bool inter = nbv >= 0;
      const bool act = inter || (nbv == NB_DIRICHLET);
      const R* Tm = WK + VOL + (s * 4 + 0) * NT * FA;
      const R* Tp = WK + VOL + (s * 4 + 1) * NT * FA;
      // general geometry: every global load of this face issued up front (one round trip)
      R Jim[9], Jip[9], wm = R(0.0), wp = R(0.0), Hp = Hm;
      if constexpr (Cf::TMA) {
        if (s == 0) mbar_wait(&mbar[lc], dd & 1);
#pragma unroll
        for (int r = 0; r < 9; ++r) Jim[r] = stg[(s * 9 + r) * n2 + p];
        wm = stg[(18 + s) * n2 + p];
        wp = wm;
        if (inter) {
#pragma unroll
          for (int r = 0; r < 9; ++r) Jip[r] = stg[(20 + s * 9 + r) * n2 + p];
          wp = stg[(38 + s) * n2 + p];
          Hp = A.Hcell[nbv];
        }
      } else if constexpr (GEO == 1) {
        const R* fm = A.fJi + ((size_t)cell * 6 + f) * 9 * n2 + p;
#pragma unroll
        for (int r = 0; r < 9; ++r) Jim[r] = __ldg(fm + r * n2);
        wm = A.nu_face[((size_t)cell * 6 + f) * n2 + p];      // nu * dA
        wp = wm;
        if (inter) {
          const R* fp = A.fJi + ((size_t)nbv * 6 + (f ^ 1)) * 9 * n2 + p;
#pragma unroll
          for (int r = 0; r < 9; ++r) Jip[r] = __ldg(fp + r * n2);
          wp = A.nu_face[((size_t)nbv * 6 + (f ^ 1)) * n2 + p];
          Hp = A.Hcell[nbv];
        }
      }
      // tangential reference derivatives of the traces (NT components)
      R tm1[NT > 0 ? NT : 1], tm2[NT > 0 ? NT : 1], tp1[NT > 0 ? NT : 1], tp2[NT > 0 ? NT : 1];
      if constexpr (NT > 0) {
        R Da[n], Db[n];
        ld_row<n>(sD + a * RS, Da);
        ld_row<n>(sD + b * RS, Db);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          R m2 = R(0.0), p2 = R(0.0);
          if (ZTR && d == 2) {
            tm1[t] = ztr[s][0];
            m2 = ztr[s][1];
          } else {
            tm1[t] = rowdot<n>(Tm + t * FA + b * RS, Da);
#pragma unroll
            for (int k = 0; k < n; ++k) m2 = fma(Db[k], Tm[t * FA + k * RS + a], m2);
          }
          tm2[t] = m2;
          if (inter) {
            tp1[t] = rowdot<n>(Tp + t * FA + b * RS, Da);
#pragma unroll
            for (int k = 0; k < n; ++k) p2 = fma(Db[k], Tp[t * FA + k * RS + a], p2);
            tp2[t] = p2;
          } else {
            tp1[t] = tm1[t];
            tp2[t] = m2;
          }
        }
      }

      R gt1[NT > 0 ? NT : 1], gt2[NT > 0 ? NT : 1];
      if constexpr (GEO == 0) {
        // ---------------- Cartesian: n = sgn e_d, J^-1 = diag(1/h)
        R num, nup, Hp = Hm;
        if constexpr (Cf::TMAC) {
          if (dd == 0 && s == 0) mbar_wait(&mbar[lc], 0);
          num = stg[f * n2 + p];
        } else if constexpr (NUF_EARLY) {
          num = nuf_m[s];
        } else {
          num = A.nu_face[((size_t)cell * 6 + f) * n2 + p];
        }
        nup = num;
        R ihp[3] = {ih[0], ih[1], ih[2]};
        if (inter && DGVV_NBCART_EARLY) {
          ihp[0] = ihq[s][0]; ihp[1] = ihq[s][1]; ihp[2] = ihq[s][2]; Hp = Hq[s];
          if constexpr (Cf::TMAC) nup = stg[(6 + f) * n2 + p];
          else if constexpr (NUF_EARLY) nup = nuf_p[s];
          else nup = A.nu_face[((size_t)nbv * 6 + (f ^ 1)) * n2 + p];
        } else if (inter) {
          const R* cg = A.cart + (size_t)nbv * CART_STRIDE;
          ihp[0] = cg[0]; ihp[1] = cg[1]; ihp[2] = cg[2]; Hp = cg[3];
          if constexpr (Cf::TMAC) nup = stg[(6 + f) * n2 + p];
          else nup = A.nu_face[((size_t)nbv * 6 + (f ^ 1)) * n2 + p];
        }
        // The SIPG flux at this face point with every per-point product folded into six scalars
        // (the same terms as PAPER.md:1055-1111 in the order of DESIGN.md §6 "K1 Cartesian flux"):
        // with sdA = sgn w_a w_b |F| and tau = pen max(H-, H+) ({{nu}}):
        //   fv_d = 2 tau dA [u_d] - (B1 du_d- + B2 du_d+),  gn_d = -B1 [u_d]      (normal component)
        //   fv_c = tau dA [u_c] - (hB1 du_c- + hB2 du_c+ + hA1_c dt_c u_d- + hA2_c dt_c u_d+),
        //   gn_c = -hB1 [u_c],  gt_c = -hA1_c [u_c]                              (tangential, c != d)
        // B1 = sdA nu- /h_d, B2 = sdA nu+ /h_d+, hB = B / 2, hA1_c = sdA nu- /(2 h_c), hA2_c = sdA nu+ /(2 h_c);
        // Laplace form: fv_c = tau dA [u_c] - (hB1 du_c- + hB2 du_c+), gn_c = -hB1 [u_c].
        const R dA = R(T.w[a]) * R(T.w[b]) * (vol * ih[d]);
        const R sdA = s ? dA : -dA;
        const R Hx = (DGVV_CARTF && DGVV_NBCART_EARLY) ? Hp : fmax(Hm, Hp);   // CARTF: Hp = max(H, H_nb)
        const R dAt = (dA * (R(0.5) * R(A.pen)) * Hx) * (num + nup);
        const R A1 = sdA * num, A2 = sdA * nup;
        const R hB1 = (R(0.5) * ih[d]) * A1, hB2 = (R(0.5) * ihp[d]) * A2;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const R jmp = um[s][c] - up[s][c];
          if (FORM == 0 && c == d) {
            const R B1 = hB1 + hB1, B2 = hB2 + hB2;
            const R t = fma(B1, dm[s][c], B2 * dp[s][c]);
            fv[s][c] = fma(dAt + dAt, jmp, -t);
            gn[s][c] = -B1 * jmp;
          } else if constexpr (FORM == 0) {
            const bool c_is_t1 = (c == t1);
            const R hA1 = (R(0.5) * ih[c]) * A1, hA2 = (R(0.5) * ih[c]) * A2;
            R t = fma(hB1, dm[s][c], hB2 * dp[s][c]);
            t = fma(hA1, c_is_t1 ? tm1[0] : tm2[0], t);
            t = fma(hA2, c_is_t1 ? tp1[0] : tp2[0], t);
            fv[s][c] = fma(dAt, jmp, -t);
            gn[s][c] = -hB1 * jmp;
            if constexpr (NT > 0) {
              if (c_is_t1) gt1[0] = -hA1 * jmp;
              else gt2[0] = -hA1 * jmp;
            }
          } else {
            fv[s][c] = fma(dAt, jmp, -fma(hB1, dm[s][c], hB2 * dp[s][c]));
            gn[s][c] = -hB1 * jmp;
          }
        }
      } else {
        // ---------------- general geometry: own / neighbour J^-1 at the face point
        // With v = J^-1 n (v_k = sum_j Ji[k][j] n_j) the physical gradient G = gx J^-1 never has
        // to be formed:  (G n)_c = gx[c].v,  (G^T n)_c = sum_k (n.gx[.][k]) Ji[k][c],  and the
        // test-side coefficients of d v_c / d xi_k are -1/2 w (jmp_c v_k + n_c (J^-1 jmp)_k)
        // (divergence form) or -1/2 w jmp_c v_k (Laplace form).
        const R sgn = s ? R(1.0) : -R(1.0);
        R nrm[3];
        {
          const R v0 = Jim[3 * d], v1 = Jim[3 * d + 1], v2 = Jim[3 * d + 2];
          const R il = sgn * rsqrt(v0 * v0 + v1 * v1 + v2 * v2);
          nrm[0] = v0 * il; nrm[1] = v1 * il; nrm[2] = v2 * il;
        }
        auto sigma_n = [&](const R (&Ji)[9], const R* gd, const R* g1, const R* g2,
                           R (&v)[3], R (&out)[NC]) {
#pragma unroll
          for (int k = 0; k < 3; ++k) v[k] = Ji[3 * k] * nrm[0] + Ji[3 * k + 1] * nrm[1] + Ji[3 * k + 2] * nrm[2];
          R gx[NC][3];
#pragma unroll
          for (int c = 0; c < NC; ++c) { gx[c][d] = gd[c]; gx[c][t1] = g1[c]; gx[c][t2] = g2[c]; }
#pragma unroll
          for (int c = 0; c < NC; ++c) out[c] = gx[c][0] * v[0] + gx[c][1] * v[1] + gx[c][2] * v[2];
          if constexpr (FORM == 0) {
            R w[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) w[k] = nrm[0] * gx[0][k] + nrm[1] * gx[1][k] + nrm[2] * gx[2][k];
#pragma unroll
            for (int c = 0; c < NC; ++c) out[c] = R(0.5) * (out[c] + w[0] * Ji[c] + w[1] * Ji[3 + c] + w[2] * Ji[6 + c]);
          } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) out[c] *= R(0.5);
          }
        };
        R spn[NC], smn[NC], vm[3];
        if (inter) {
          R vp[3];
          sigma_n(Jip, dp[s], tp1, tp2, vp, spn);
        }
        sigma_n(Jim, dm[s], tm1, tm2, vm, smn);
        if (!inter) {
#pragma unroll
          for (int c = 0; c < NC; ++c) spn[c] = smn[c];
        }
        const R tau = R(A.pen) * fmax(Hm, Hp) * R(0.5) * (wm + wp);
        R jmp[NC], jn = R(0.0);
#pragma unroll
        for (int c = 0; c < NC; ++c) jmp[c] = um[s][c] - up[s][c];
        R q[3] = {R(0.0), R(0.0), R(0.0)};
        if constexpr (FORM == 0) {
#pragma unroll
          for (int c = 0; c < NC; ++c) jn += jmp[c] * nrm[c];
#pragma unroll
          for (int k = 0; k < 3; ++k) q[k] = Jim[3 * k] * jmp[0] + Jim[3 * k + 1] * jmp[1] + Jim[3 * k + 2] * jmp[2];
        }
        const R hw = -R(0.5) * wm;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const R pv = (FORM == 0) ? (jmp[c] + nrm[c] * jn) : jmp[c];
          fv[s][c] = -(wm * smn[c] + wp * spn[c]) + tau * pv;
          R gk[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) gk[k] = (FORM == 0) ? hw * (jmp[c] * vm[k] + nrm[c] * q[k]) : hw * jmp[c] * vm[k];
          gn[s][c] = gk[d];
          gt1[c] = gk[t1];
          gt2[c] = gk[t2];
        }
      }
      if (!act) {
#pragma unroll
        for (int c = 0; c < NC; ++c) { fv[s][c] = R(0.0); gn[s][c] = R(0.0); }
        if constexpr (NT > 0) {
#pragma unroll
          for (int t = 0; t < NT; ++t) { gt1[t] = R(0.0); gt2[t] = R(0.0); }
        }
      }
      if constexpr (CONV) {
        // f4 (fused): upwind flux of the convective term, a value term of this side's test
        // functions: min({{w}}.n, 0) dA (u+ - u-) on interior/periodic faces (readings F4a/F4b),
        // with the stored face factor (0 where this side is outflow and on boundary faces)
        const R cf = R(A.alpha_c) * __ldg(A.wface + ((size_t)cell * 6 + f) * n2 + p);
#pragma unroll
        for (int c = 0; c < NC; ++c) fv[s][c] = fma(cf, up[s][c] - um[s][c], fv[s][c]);
      }
      if constexpr (NT > 0) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          WK[VOL + ((s * 4 + 2) * NT + t) * FA + b * RS + a] = gt1[t];
          WK[VOL + ((s * 4 + 3) * NT + t) * FA + a * RS + b] = gt2[t];
        }
      }
    }
    // value coefficient at each face node = fv + transposed tangential contributions
    if constexpr (NT > 0) {
      __syncthreads();
      if constexpr (Cf::TMA) {
        if (dd < 2 && p == 0) stage_issue(dd == 0 ? 0 : 1, nbf);   // stage is free: next direction
      }
      R DTa[n], DTb[n];
      ld_row<n>(sDT + a * RS, DTa);
      ld_row<n>(sDT + b * RS, DTb);
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const int c = (GEO == 1) ? t : d;
          fv[s][c] += rowdot<n>(WK + VOL + ((s * 4 + 2) * NT + t) * FA + b * RS, DTa) +
                      rowdot<n>(WK + VOL + ((s * 4 + 3) * NT + t) * FA + a * RS, DTb);
        }
    }

    // extrapolate both faces' coefficients along the normal line into the cell
    if (NT == 0 && d == 1) __syncthreads();   // x-fold reads of Y are complete
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      R add[n];
#pragma unroll
      for (int i = 0; i < n; ++i)
        add[i] = R(T.l0[i]) * fv[0][c] + R(T.d0[i]) * gn[0][c] + R(T.l1[i]) * fv[1][c] + R(T.d1[i]) * gn[1][c];
      if (d == 2) {
#pragma unroll
        for (int i = 0; i < n; ++i) y[c][i] += add[i];
      } else {
        st_row<n>(WK + c * CST + b * PS + a * RS, add);
      }
    }
    if (d != 2) {
      __syncthreads();
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int z = 0; z < n; ++z)
          y[c][z] += (d == 0) ? WK[c * CST + z * PS + b * RS + a] : WK[c * CST + z * PS + a * RS + b];
    }
  }

  // =============================================================== epilogue
  if constexpr (MASS) {                 // Helmholtz mass term: + mass * JxW * u (diagonal M)
#pragma unroll
    for (int z = 0; z < n; ++z) {
      R mjw;
      if constexpr (GEO == 0) mjw = R(A.mass) * R(T.w[a]) * R(T.w[b]) * R(T.w[z]) * vol;
      else mjw = R(A.mass) * A.jxw[(size_t)cell * n3 + z * n2 + p];
#pragma unroll
      for (int c = 0; c < NC; ++c) y[c][z] += mjw * su[c * CST + z * PS + b * RS + a];
    }
  }
  if (active) {
    // the epilogue mode is uniform: branch once, not per element (per-element tests compiled to a
    // jump table per store, ncu: 12 indirect branches per thread)
    const size_t off = (size_t)cell * NC * n3 + p;
    if (A.mode == MODE_APPLY) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int z = 0; z < n; ++z) A.dst[off + c * n3 + z * n2] = y[c][z];
    } else if (A.mode == MODE_RESID) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int z = 0; z < n; ++z) {
          const size_t i = off + c * n3 + z * n2;
          A.dst[i] = __ldg(A.b + i) - y[c][z];
        }
    } else {
      // every load of the update (b, D^-1, d) is issued before the first store: d is read and
      // written in place, so a load of d placed after a store to d / x_out in program order cannot
      // be hoisted above it (possible aliasing) and the NC * n iterations would each pay a full
      // DRAM round trip (measured: C5 Chebyshev apply 4.5 ms against 2.7 ms for the plain apply)
      const R cr = R(A.c_r), crho = R(A.c_rho);
      R bv[NC][n], dv[NC][n], dd[NC][n];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int z = 0; z < n; ++z) {
          const size_t i = off + c * n3 + z * n2;
          bv[c][z] = __ldg(A.b + i);
          dv[c][z] = __ldg(A.dinv + i);
        }
      if (crho != R(0.0)) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int z = 0; z < n; ++z) dd[c][z] = crho * A.dvec[off + c * n3 + z * n2];
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int z = 0; z < n; ++z) dd[c][z] = R(0.0);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int z = 0; z < n; ++z) {
          const size_t i = off + c * n3 + z * n2;
          const R r = bv[c][z] - y[c][z];
          const R dn = cr * dv[c][z] * r + dd[c][z];
          A.dvec[i] = dn;
          A.xout[i] = su[c * CST + z * PS + b * RS + a] + dn;
        }
    }
  }
}

}  // namespace dgvv
