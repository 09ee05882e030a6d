// Batched compact-WY block reflector application (see wy.cuh).
//
// Template NB in {32, 64} (reflectors per block), 8*NB/32 warps per CTA.
// One CTA owns one (block, TN-column tile) and streams the rows in RC-row
// chunks through a cp.async ring (full/empty mbarriers, no CTA barrier per
// chunk), twice: phase 1 accumulates
// W = V^T C (NB x TN) with the k (row) dimension split over two warp groups
// (each warp: 2 x 4 mma tiles, 6 fragment loads per 8 DMMA), phase 2 forms
// W' = op(T) W (T read through L1/L2), phase 3 updates C -= V W' with W'
// held in registers and stores the accumulators straight to global memory.
// NB = 64 doubles the arithmetic intensity per pass over C (4*NB flops per
// 24 bytes), which moves the update from the HBM roof to the DMMA roof.
#include "wy.cuh"

namespace {

constexpr int TN = 64;            // C columns per CTA
constexpr int RC = 32;            // rows per staged chunk
// T_j is read through L1/L2, not staged in shared memory (measured on cfg4,
// wy<64>, 2 filters: staged 79.8 ms, through L1/L2 75.3: the 32 KB go to L1).
// Ring stages, measured on cfg4: wy<64> 4 stages 1.4% faster than 3 (296.9 vs
// 301.1 ms per two filters); wy<32>, 2 filters: 3 stages 30.3 ms, 2 stages
// 38.8, 4 stages 42.3.
constexpr int WY_STAGES64 = 4, WY_STAGES32 = 3;
// Measured and not kept (round 2): warp-uniform skips of the n-tiles past a
// tile's last column (the 32-column panel-local updates use half of a 64-column
// tile): wy<64> 75.3 -> 90.8 ms and wy<32> 30.3 -> 33.2 ms per two filters
// (the branches around the unrolled MMA loops cost more than the idle tiles).
template <int NB>
constexpr int stages_for() { return NB == 64 ? WY_STAGES64 : WY_STAGES32; }
constexpr int LDS = RC + 4;       // padded column length of a staged chunk
constexpr int LDW = TN + 4;       // padded row length of W

template <int NB>
struct Cfg {
  static constexpr int NW = 8 * NB / 32;
  static constexpr int NT = NW * 32;
  static constexpr int STAGES = stages_for<NB>();
  static constexpr size_t smem = (size_t)(STAGES * NB * LDS + STAGES * TN * LDS + NB * LDW) * 8;
};

template <int NB>
__device__ __forceinline__ void load_chunk(const double* __restrict__ V, int vld, const double* __restrict__ C,
                                           int cld, int ncol, int rbase, double* vs, double* cs) {
  constexpr int NT = Cfg<NB>::NT;
  for (int p = threadIdx.x; p < NB * (RC / 2); p += NT) {
    const int col = p / (RC / 2), rr = (p % (RC / 2)) * 2, row = rbase + rr;
    double* dst = vs + col * LDS + rr;
    if (row < vld) fl::cp_async16(dst, V + (int64_t)col * vld + row);
    else fl::cp_async16_zero(dst, V);
  }
  for (int p = threadIdx.x; p < TN * (RC / 2); p += NT) {
    const int col = p / (RC / 2), rr = (p % (RC / 2)) * 2, row = rbase + rr;
    double* dst = cs + col * LDS + rr;
    if (col < ncol && row < cld) fl::cp_async16(dst, C + (int64_t)col * cld + row);
    else fl::cp_async16_zero(dst, C);
  }
}

// unit lower-trapezoidal structure of V's first NB rows: chunk rows base..base+RC
template <int NB>
__device__ __forceinline__ void mask_unit(double* vs, int base) {
  constexpr int NT = Cfg<NB>::NT;
  for (int p = threadIdx.x; p < NB * RC; p += NT) {
    const int col = p / RC, rr = p % RC, row = base + rr;
    if (row <= col) vs[col * LDS + rr] = (row == col) ? 1.0 : 0.0;
  }
}

template <int NB>
__global__ void __launch_bounds__(Cfg<NB>::NT, (NB == 32 ? 2 : 1)) wy_apply_kernel(fl::WyArgs a) {
  constexpr int NW = Cfg<NB>::NW;
  constexpr int STAGES = Cfg<NB>::STAGES;
  extern __shared__ double sm[];
  double* Vs = sm;                            // [STAGES][NB][LDS]
  double* Cs = Vs + STAGES * NB * LDS;        // [STAGES][TN][LDS]
  double* Ws = Cs + STAGES * TN * LDS;        // [NB][LDW]

  int j, c0;
  if (a.tiles) {
    j = a.tiles[2 * blockIdx.x];
    c0 = a.tiles[2 * blockIdx.x + 1];
  } else {
    j = blockIdx.x / a.tiles_per_block;
    c0 = (blockIdx.x % a.tiles_per_block) * TN;
  }
  const int mj = a.m[j];
  const int r0 = a.row0;
  const int ncol = min(TN, (a.ncols ? a.ncols[j] - a.ncols_sub : a.ncols_const) - c0);
  if (mj <= r0 || ncol <= 0) return;
  const int vld = a.vld ? a.vld[j] : a.vld_const, cld = a.cld ? a.cld[j] : a.cld_const;
  const double* V = a.V + (a.voff ? a.voff[j] : j * a.vstride) + a.v_col0 * (int64_t)vld;
  double* C = a.C + (a.coff ? a.coff[j] : j * a.cstride) + (a.c_col0 + c0) * (int64_t)cld;
  const double* Cin = a.Csrc ? a.Csrc + (C - a.C) : C;  // where C is read from
  const int nchunks = (mj - r0 + RC - 1) / RC;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;

  const double* Tg = a.T + (int64_t)j * a.tstride;  // read through L1/L2 in phase 2

  auto stage_v = [&](int s) { return Vs + s * NB * LDS; };
  auto stage_c = [&](int s) { return Cs + s * TN * LDS; };

  // ---------------- phase 1: W = V^T C ----------------
  constexpr int MB = NB / 16;  // m-tile pairs
  const int kg = w / (NW / 2), wl = w % (NW / 2);
  const int mb = wl % MB, nbk = wl / MB;
  double acc[2][4][2];
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int n = 0; n < 4; ++n) acc[mi][n][0] = acc[mi][n][1] = 0.0;
  // full/empty mbarrier ring (no CTA barrier per chunk): chunk G of the
  // kernel (phase 1 then phase 3 numbering) uses stage G % STAGES for the
  // (G / STAGES)-th time; both barriers of the stage complete the phase of
  // parity (G / STAGES) & 1 for it
  __shared__ uint64_t full[STAGES], empty[STAGES];
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      fl::mbar_init(&full[i], Cfg<NB>::NT);
      fl::mbar_init(&empty[i], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto load = [&](int ch, int G) {
    const int st = G % STAGES;
    load_chunk<NB>(V, vld, Cin, cld, ncol, r0 + ch * RC, stage_v(st), stage_c(st));
    fl::cp_async_arrive(&full[st]);
  };
  // chunk G's data: wait, then the unit-trapezoid mask on the first chunks
  auto acquire = [&](int ch, int G) {
    const int st = G % STAGES;
    fl::mbar_wait(&full[st], (G / STAGES) & 1);
    if (ch * RC < NB) {  // (every copy of the stage has landed once full[st] completes)
      mask_unit<NB>(stage_v(st), ch * RC);
      __syncthreads();
    }
  };
  // leave chunk G's stage and refill it with chunk ch + STAGES - 1 of this pass
  auto release = [&](int ch, int G, int n, int Gbase) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) fl::mbar_arrive(&empty[G % STAGES]);
    const int nx = ch + STAGES - 1;
    if (nx < n) {
      const int Gn = Gbase + nx, Gp = Gn - STAGES;  // previous user of the stage
      if (Gp >= 0) fl::mbar_wait(&empty[Gn % STAGES], (Gp / STAGES) & 1);
      load(nx, Gn);
    }
  };
  auto prologue = [&](int n, int Gbase) {
    for (int c = 0; c < STAGES - 1 && c < n; ++c) {
      const int Gn = Gbase + c, Gp = Gn - STAGES;
      if (Gp >= 0) fl::mbar_wait(&empty[Gn % STAGES], (Gp / STAGES) & 1);
      load(c, Gn);
    }
  };

  prologue(nchunks, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    acquire(ch, ch);
    const double* vs = stage_v(ch % STAGES);
    const double* cs = stage_c(ch % STAGES);
#pragma unroll
    for (int s = kg; s < RC / 4; s += 2) {
      const int k0 = 4 * s;
      double av[2], bv[4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) av[mi] = vs[((2 * mb + mi) * 8 + g) * LDS + k0 + t];
#pragma unroll
      for (int n = 0; n < 4; ++n) bv[n] = cs[((4 * nbk + n) * 8 + g) * LDS + k0 + t];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int n = 0; n < 4; ++n) fl::dmma(acc[mi][n][0], acc[mi][n][1], av[mi], bv[n]);
    }
    release(ch, ch, nchunks, 0);
  }
  // phase 3's first chunks stream in while W is reduced and multiplied by T
  prologue(nchunks, nchunks);
  if (kg == 1) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const int row = (2 * mb + mi) * 8 + g, col = (4 * nbk + n) * 8 + 2 * t;
        Ws[row * LDW + col] = acc[mi][n][0];
        Ws[row * LDW + col + 1] = acc[mi][n][1];
      }
  }
  __syncthreads();
  if (kg == 0) {
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        const int row = (2 * mb + mi) * 8 + g, col = (4 * nbk + n) * 8 + 2 * t;
        Ws[row * LDW + col] += acc[mi][n][0];
        Ws[row * LDW + col + 1] += acc[mi][n][1];
      }
  }
  __syncthreads();

  // ---------------- phase 2: W <- op(T) W  (NB x 64: 4 tiles per warp) ----------------
  {
    const int mt = w % (NB / 8), ntb = (w / (NB / 8)) * 4;
    double p2[4][2];
#pragma unroll
    for (int n = 0; n < 4; ++n) p2[n][0] = p2[n][1] = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < NB; k0 += 4) {
      const int ar = mt * 8 + g, ac = k0 + t;
      const double av = __ldg(a.transT ? Tg + ar * NB + ac : Tg + ac * NB + ar);  // op(T)[ar][ac]
#pragma unroll
      for (int n = 0; n < 4; ++n) fl::dmma(p2[n][0], p2[n][1], av, Ws[(k0 + t) * LDW + (ntb + n) * 8 + g]);
    }
    __syncthreads();
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      Ws[(mt * 8 + g) * LDW + (ntb + n) * 8 + 2 * t] = p2[n][0];
      Ws[(mt * 8 + g) * LDW + (ntb + n) * 8 + 2 * t + 1] = p2[n][1];
    }
    __syncthreads();
  }

  // ---------------- phase 3: C -= V W' ----------------
  constexpr int NN = 32 / NW;  // n-tiles per warp: 4 (NB 32) or 2 (NB 64)
  const int mrow = (w % 4) * 8, ncb = (w / 4) * NN;
  double bw[NB / 4][NN];
#pragma unroll
  for (int k = 0; k < NB / 4; ++k)
#pragma unroll
    for (int n = 0; n < NN; ++n) bw[k][n] = Ws[(4 * k + t) * LDW + (ncb + n) * 8 + g];
  for (int ch = 0; ch < nchunks; ++ch) {
    const int G = nchunks + ch;
    const int rbase = r0 + ch * RC;
    acquire(ch, G);
    const double* vs = stage_v(G % STAGES);
    const double* cs = stage_c(G % STAGES);
    double c[NN][2];
#pragma unroll
    for (int n = 0; n < NN; ++n) {
      const int row = mrow + g, col = (ncb + n) * 8 + 2 * t;
      c[n][0] = cs[col * LDS + row];
      c[n][1] = cs[(col + 1) * LDS + row];
    }
#pragma unroll
    for (int k = 0; k < NB / 4; ++k) {
      const double av = -vs[(4 * k + t) * LDS + mrow + g];
#pragma unroll
      for (int n = 0; n < NN; ++n) fl::dmma(c[n][0], c[n][1], av, bw[k][n]);
    }
    // direct stores from the accumulators (no shared-memory round trip)
    {
      const int row = rbase + mrow + g;
      if (row < mj) {
#pragma unroll
        for (int n = 0; n < NN; ++n) {
          const int col = (ncb + n) * 8 + 2 * t;
          if (col < ncol) C[(int64_t)col * cld + row] = c[n][0];
          if (col + 1 < ncol) C[(int64_t)(col + 1) * cld + row] = c[n][1];
        }
      }
    }
    release(ch, G, nchunks, nchunks);
  }
}

template <int NB>
int launch(const fl::WyArgs& a, cudaStream_t s) {
  static unsigned long long attr = 0;
  if (fl::first_on_device(attr)) {
    FL_CUDA(cudaFuncSetAttribute(wy_apply_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)Cfg<NB>::smem));
  }
  wy_apply_kernel<NB><<<a.ntiles, Cfg<NB>::NT, Cfg<NB>::smem, s>>>(a);
  FL_CHECK_LAUNCH();
  return FL_OK;
}

}  // namespace

namespace fl {
int wy_apply(const WyArgs& a, cudaStream_t s) { return wy_apply_nb(a, 32, s); }
int wy_apply_nb(const WyArgs& a, int nb, cudaStream_t s) {
  if (a.ntiles == 0) return FL_OK;
  if (nb == 64) return launch<64>(a, s);
  if (nb == 32) return launch<32>(a, s);
  return FL_ERR_INVALID;
}
int wy_nb() { return 32; }
int wy_tn() { return TN; }
}  // namespace fl

// Diagnostic entry point: one launch of the block reflector kernel over
// caller-built tables (all device pointers), for kernel-level tests.
extern "C" int fl_dev_wy_apply(const double* V, const int64_t* voff, const int32_t* vld, double* C,
                               const int64_t* coff, const int32_t* cld, const int32_t* m, const double* T,
                               int64_t tstride, int32_t nb, int32_t row0, int32_t transT, const int32_t* ncols,
                               const int32_t* tiles, int32_t ntiles, void* stream) {
  fl::WyArgs a{};
  a.V = V;
  a.voff = voff;
  a.vld = vld;
  a.C = C;
  a.coff = coff;
  a.cld = cld;
  a.m = m;
  a.T = T;
  a.tstride = tstride;
  a.row0 = row0;
  a.transT = transT;
  a.ncols = ncols;
  a.tiles = tiles;
  a.ntiles = ntiles;
  return fl::wy_apply_nb(a, nb, (cudaStream_t)stream);
}
