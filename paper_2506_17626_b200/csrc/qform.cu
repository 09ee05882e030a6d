// K2c, fused form: Q_j = Q0_j [Q1_j; 0] with ONE pass over Q per 64-reflector
// block of Q0_j instead of two.
//
// Q0_j = H_0 .. H_{K-1} is applied to C = [Q1_j; 0] block by block in reverse
// (b = nb-1 .. 0), each block in compact-WY form C -= V_b T_b (V_b^T C). The
// two-pass kernel (wy.cu) streams C once for W_b = V_b^T C and once for the
// update. Here one CTA owns a 64-column tile of C for the whole sequence, so
// the update pass of block b also accumulates W_{b-1} = V_{b-1}^T C from the
// freshly updated rows (rows >= 64(b-1); rows 64(b-1)..64b-1 are read by the
// same pass since V_b vanishes there). The sequence is
//     B(nb-1) ; A(nb-1)+B(nb-2) ; ... ; A(1)+B(0) ; A(0)
// (A = apply, B = accumulate), nb + 1 passes over C instead of 2 nb, and the
// first one only reads rows 64(nb-1)..K-1 because C is zero below row K
// until A(nb-1) runs (which also skips loading those rows).
//
// Every product is mma.sync m8n8k4 f64 (DMMA), as in wy.cu. Chunks of 32
// rows of [V_{b-1} | V_b] (128 columns) and C (64 columns) are staged with
// 16-byte cp.async in a 3-stage ring. Between passes the ring's memory holds
// W and T_{b-1} for W' = T_{b-1} W, which is kept in shared memory behind
// the ring for the next pass's update. (Measured alternative, not kept:
// warps split into an update group and an accumulate group one chunk apart,
// one barrier per chunk: 69% DMMA pipe activity but 94.6 vs 91.3 ms.)
#include "wy.cuh"

namespace {

constexpr int NB = 64;    // reflectors per block
constexpr int TN = 64;    // C columns per CTA
// CTA shape: QF_NW warps, 2 NW-row chunks (every phase-A warp owns one
// m-tile x two n-tiles), QF_MINB CTAs per SM, QF_STAGES ring stages.
// Measured on cfg4 (ncu, one filter): 16 warps / 3 stages 89.1 ms, 4 stages
// 89.7 ms, 8 warps at two CTAs per SM 101.8 ms. With the mbarrier ring: a
// 32 KB shared buffer for T prefetched during the pass 85.7 vs 78.2 ms (every
// extra KB of shared memory is taken from L1, which this kernel needs). Without the per-chunk
// barriers (incorrect, timing only) 72 ms: the barriers, not the loads or
// shared-memory bandwidth, hold the DMMA pipe near 68% busy.
constexpr int QF_NW = 16, QF_MINB = 1, QF_STAGES = 3;
constexpr int NW = QF_NW, NT = NW * 32;
constexpr int RC = 2 * NW;  // rows per staged chunk
constexpr int QF_PAD = 4;
constexpr int LDS = RC + QF_PAD; // 4: = 4 mod 16, conflict-free 8-byte fragment loads
// (measured on cfg4: pad 4 78.2 ms, pad 2 — 2-way conflicts, ring small enough
// for the 164 KB shared-memory configuration — 80.4, pad 0 128 ms)
// (measured: an unpadded layout with the row index XOR 4 (col mod 4) —
// conflict-free as well, 11% less shared memory — 87.4 vs 78.2 ms on cfg4)
constexpr int LDW = TN + 4;
constexpr int MT = RC / 8;            // m-tiles per chunk
constexpr int BNN = 64 / NW / 2;     // phase-B warp tile: 2 m-tiles x BNN n-tiles
constexpr int SLOTS = TN * (RC / 2) / NT;  // 16-byte staging slots per thread per operand
static_assert(SLOTS * NT == TN * (RC / 2), "staging slots");
static_assert(4 * MT == NW, "phase-A tiling");
constexpr int STAGES = QF_STAGES;
constexpr int VST = 2 * NB * LDS;  // doubles per V stage: V_{b-1} columns 0..63, V_b columns 64..127
constexpr int CST = TN * LDS;
constexpr size_t RING = (size_t)STAGES * (VST + CST) * sizeof(double);
constexpr size_t SMEM = RING;
static_assert((size_t)(2 * NB * LDW) * sizeof(double) <= RING, "W and W' fit in the ring");

struct QfArgs {
  const double* V;       // factored A store (reflectors below the diagonal)
  const int64_t* voff;
  const int32_t* vld;
  const int32_t* m;
  double* C;             // Q store, holding [Q1; 0] on entry
  const int64_t* coff;
  const int32_t* cld;
  const int32_t* rank;   // columns of C per block
  const double* T64;     // (J, K/64, 64, 64) column-major upper-triangular T_b
  int K;
  int tiles_per_block;
};

__global__ void __launch_bounds__(NT, QF_MINB) qform_kernel(QfArgs a) {
  extern __shared__ double sm[];
  double* Vs = sm;                      // [STAGES][128][LDS]
  double* Cs = Vs + STAGES * VST;       // [STAGES][64][LDS]
  double* Ws = sm;                      // between passes: W [64][LDW]
  double* Wp = sm + NB * LDW;           //                 W' = T W [64][LDW]

  const int j = blockIdx.x / a.tiles_per_block;
  const int c0 = (blockIdx.x % a.tiles_per_block) * TN;
  const int mj = a.m[j];
  const int ncol = min(TN, a.rank[j] - c0);
  if (ncol <= 0 || mj <= 0) return;
  const int K = a.K;
  // null offset / ld tables: dense (J, K, K) stores, ld K (the QRCP factor R0 and Q1)
  const int vld = a.vld ? a.vld[j] : K, cld = a.cld ? a.cld[j] : K;
  const double* V = a.V + (a.voff ? a.voff[j] : (int64_t)j * K * K);
  double* C = a.C + (a.coff ? a.coff[j] : (int64_t)j * K * K) + (int64_t)c0 * cld;
  const double* Tj = a.T64 + (int64_t)j * (K / NB) * NB * NB;
  const int nact = min(K / NB, (mj + NB - 1) / NB);  // blocks with reflectors
  if (nact <= 0) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;

  // this thread's (column, row pair) staging slots of a 64 x RC tile
  int scol[SLOTS], srr[SLOTS];
#pragma unroll
  for (int it = 0; it < SLOTS; ++it) {
    const int p = threadIdx.x + it * NT;
    scol[it] = p / (RC / 2);
    srr[it] = (p % (RC / 2)) * 2;
  }

  // Register blocking sized for shared-memory traffic (both phases read
  // their operands from the ring): phase A (C -= V W', 32 x 64) warp tile =
  // one m-tile x two n-tiles with W' held in registers for the whole pass, so
  // a V fragment feeds two DMMAs and W' is never re-read (128 B of shared
  // loads per DMMA); phase B (W = V^T C, 64 x 64) warp tile = 2 x 2 tiles
  // over all of the chunk's rows (256 B per DMMA, no cross-warp reduction).
  const int am = w % MT, an = 2 * (w / MT);
  const int bm = 2 * (w % 4), bn = BNN * (w / 4);
  double bw[NB / 4][2];  // W'(4k + t, 8 (an + n) + g)
  double acc[2][BNN][2];

  __shared__ uint64_t full[STAGES], empty[STAGES];
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      fl::mbar_init(&full[i], NT);   // one cp.async arrival per thread
      fl::mbar_init(&empty[i], NW);  // one arrival per warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  int G0 = 0;

  int bA = -1, bB = nact - 1;
  for (;;) {
    const bool doA = bA >= 0, doB = bB >= 0;
    const int rlo = doB ? NB * bB : NB * bA;
    const int rhi = doA ? mj : min(mj, K);
    // C rows >= K are zero until the first update has run
    const int cz = (bA == nact - 1 || !doA) ? K : cld;
    const int nch = (rhi - rlo + RC - 1) / RC;
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int n = 0; n < BNN; ++n) acc[mi][n][0] = acc[mi][n][1] = 0.0;

    // every thread stages its slots of chunk ch into ring stage st and arrives
    // on full[st] when its copies land (out-of-range rows are zero-filled by
    // the same async unit, so one wait on full[st] covers all of the stage)
    auto load = [&](int ch, int st) {
      const int rbase = rlo + ch * RC;
      double* vs = Vs + st * VST;
      double* cs = Cs + st * CST;
#pragma unroll
      for (int it = 0; it < SLOTS; ++it) {
        const int col = scol[it], rr = srr[it], row = rbase + rr;
        if (doB) {
          double* d = vs + col * LDS + rr;
          if (row < vld) fl::cp_async16(d, V + (int64_t)(NB * bB + col) * vld + row);
          else fl::cp_async16_zero(d, V);
        }
        if (doA) {
          double* d = vs + (NB + col) * LDS + rr;
          if (row < vld) fl::cp_async16(d, V + (int64_t)(NB * bA + col) * vld + row);
          else fl::cp_async16_zero(d, V);
        }
        double* d = cs + col * LDS + rr;
        if (col < ncol && row < cz && row < cld) fl::cp_async16(d, C + (int64_t)col * cld + row);
        else fl::cp_async16_zero(d, C);
      }
      fl::cp_async_arrive(&full[st]);
    };

    // Chunks are numbered across passes (G); chunk G uses stage G % STAGES
    // for the (G / STAGES)-th time, so both barriers of that stage complete
    // their phase of parity (G / STAGES) & 1 for it. No CTA barrier per
    // chunk: a warp waits for its chunk's data (full) and, before refilling a
    // stage, for every warp to have left it (empty), which is a chunk later.
    for (int c = 0; c < STAGES - 1 && c < nch; ++c) load(c, (G0 + c) % STAGES);
    for (int ch = 0; ch < nch; ++ch) {
      const int G = G0 + ch, st = G % STAGES;
      const int rbase = rlo + ch * RC;
      fl::mbar_wait(&full[st], (G / STAGES) & 1);
      double* vs = Vs + st * VST;
      double* cs = Cs + st * CST;
      // unit lower-trapezoidal structure: V_b's diagonal starts at row 64 b
      const bool mB = doB && rbase < NB * bB + NB, mA = doA && rbase < NB * bA + NB;
      if (mB || mA) {
        for (int p = threadIdx.x; p < NB * RC; p += NT) {
          const int col = p / RC, rr = p % RC;
          if (mB) {
            const int rel = rbase + rr - NB * bB;
            if (rel <= col) vs[col * LDS + rr] = (rel == col) ? 1.0 : 0.0;
          }
          if (mA) {
            const int rel = rbase + rr - NB * bA;
            if (rel <= col) vs[(NB + col) * LDS + rr] = (rel == col) ? 1.0 : 0.0;
          }
        }
        __syncthreads();
      }
      // ---- A: C -= V_b W' on this chunk (rows above 64 b are untouched) ----
      if (doA && rbase + RC > NB * bA) {
        const double* vb = vs + NB * LDS;
        double c[2][2];
        const int row = am * 8 + g;
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const int col = (an + n) * 8 + 2 * t;
          c[n][0] = cs[col * LDS + row];
          c[n][1] = cs[(col + 1) * LDS + row];
        }
#pragma unroll
        for (int k = 0; k < NB / 4; ++k) {
          const double av = -vb[(4 * k + t) * LDS + row];
#pragma unroll
          for (int n = 0; n < 2; ++n) fl::dmma(c[n][0], c[n][1], av, bw[k][n]);
        }
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          const int col = (an + n) * 8 + 2 * t;
          cs[col * LDS + row] = c[n][0];
          cs[(col + 1) * LDS + row] = c[n][1];
          if (rbase + row < mj) {
            if (col < ncol) C[(int64_t)col * cld + rbase + row] = c[n][0];
            if (col + 1 < ncol) C[(int64_t)(col + 1) * cld + rbase + row] = c[n][1];
          }
        }
        // B below reads only C columns written by the 4 warps of this warp's
        // group (an == bn): a named barrier over those 128 threads
        if (doB) asm volatile("bar.sync %0, 128;\n" ::"r"(1 + w / 4) : "memory");
      }
      // ---- B: W_{b-1} += V_{b-1}^T C on the (updated) chunk ----
      if (doB) {
#pragma unroll
        for (int s = 0; s < RC / 4; ++s) {
          const int k0 = 4 * s;
          double av[2], bv[BNN];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) av[mi] = vs[((bm + mi) * 8 + g) * LDS + k0 + t];
#pragma unroll
          for (int n = 0; n < BNN; ++n) bv[n] = cs[((bn + n) * 8 + g) * LDS + k0 + t];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int n = 0; n < BNN; ++n) fl::dmma(acc[mi][n][0], acc[mi][n][1], av[mi], bv[n]);
        }
      }
      __syncwarp();
      if (lane == 0) fl::mbar_arrive(&empty[st]);
      if (ch + STAGES - 1 < nch) {
        // stage of chunk ch + STAGES - 1 = stage of chunk ch - 1 (free before
        // this pass when ch == 0: the passes are separated by a CTA barrier)
        const int sn = (G + STAGES - 1) % STAGES;
        if (ch >= 1) fl::mbar_wait(&empty[sn], ((G - 1) / STAGES) & 1);
        load(ch + STAGES - 1, sn);
      }
    }
    G0 += nch;
    if (!doB) break;

    // ---- between passes: W' = T_{b-1} W in the ring's memory (T from L2),
    //      then W' fragments to registers ----
    fl::cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int n = 0; n < BNN; ++n) {
        const int row = (bm + mi) * 8 + g, col = (bn + n) * 8 + 2 * t;
        Ws[row * LDW + col] = acc[mi][n][0];
        Ws[row * LDW + col + 1] = acc[mi][n][1];
      }
    __syncthreads();
    {
      constexpr int N2 = 64 / NW;  // n-tiles of W' per warp
      const int mt = w % 8, ntb = (w / 8) * N2;
      const double* Tb = Tj + (int64_t)bB * NB * NB;
      double p2[N2][2];
#pragma unroll
      for (int n = 0; n < N2; ++n) p2[n][0] = p2[n][1] = 0.0;
#pragma unroll 4
      for (int k0 = 0; k0 < NB; k0 += 4) {
        const double av = __ldg(Tb + (k0 + t) * NB + mt * 8 + g);  // T[mt*8+g][k0+t]
#pragma unroll
        for (int n = 0; n < N2; ++n) fl::dmma(p2[n][0], p2[n][1], av, Ws[(k0 + t) * LDW + (ntb + n) * 8 + g]);
      }
#pragma unroll
      for (int n = 0; n < N2; ++n) {
        Wp[(mt * 8 + g) * LDW + (ntb + n) * 8 + 2 * t] = p2[n][0];
        Wp[(mt * 8 + g) * LDW + (ntb + n) * 8 + 2 * t + 1] = p2[n][1];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NB / 4; ++k)
#pragma unroll
      for (int n = 0; n < 2; ++n) bw[k][n] = Wp[(4 * k + t) * LDW + (an + n) * 8 + g];
    __syncthreads();  // the ring is reloaded by the next pass
    bA = bB;
    --bB;
  }
}

}  // namespace

namespace fl {
// Q (blocks at coff/cld, holding [Q1; 0]) <- Q0 Q for every block; K % 64 == 0.
int qform_fused(const double* V, const int64_t* voff, const int32_t* vld, const int32_t* m, double* C,
                const int64_t* coff, const int32_t* cld, const int32_t* rank, const double* T64, int K, int J,
                cudaStream_t s) {
  if (K % NB) return FL_ERR_INVALID;
  static unsigned long long attr = 0;
  if (fl::first_on_device(attr)) {
    FL_CUDA(cudaFuncSetAttribute(qform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  }
  QfArgs a{V, voff, vld, m, C, coff, cld, rank, T64, K, (K + TN - 1) / TN};
  qform_kernel<<<J * a.tiles_per_block, NT, SMEM, s>>>(a);
  FL_CHECK_LAUNCH();
  return FL_OK;
}
}  // namespace fl

// Diagnostic entry point: one fused K2c launch over caller-built block tables
// (device pointers), for kernel-level tests.
extern "C" int fl_dev_qform(const double* V, const int64_t* voff, const int32_t* vld, const int32_t* m, double* C,
                            const int64_t* coff, const int32_t* cld, const int32_t* rank, const double* T64,
                            int32_t K, int32_t nblocks, void* stream) {
  if (nblocks == 0) return FL_OK;
  if (!voff || !vld || !coff || !cld) return FL_ERR_INVALID;
  return fl::qform_fused(V, voff, vld, m, C, coff, cld, rank, T64, K, nblocks, (cudaStream_t)stream);
}
