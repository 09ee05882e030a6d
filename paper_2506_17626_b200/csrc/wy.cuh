// Batched compact-WY block reflector application on FP64 tensor cores.
//
//   C_j[row0:m_j, cols] -= V_j[row0:m_j, 0:NB] * op(T_j) * V_j[row0:m_j, 0:NB]^T * C_j[row0:m_j, cols]
//
// V_j is the unit lower-trapezoidal panel of NB Householder vectors whose
// unit diagonal starts at row0 (entries above it are ignored), T_j the NB x NB
// upper-triangular WY factor (dlarft), op(T) = T^T for Q^T C (trailing update
// of a factorisation) and T for Q C (forming Q). One CTA owns one (block,
// TN-column tile) and streams the rows in RC-row chunks through shared
// memory (cp.async, double buffered) twice: once for W = V^T C, once for
// C -= V (op(T) W). All products are mma.sync m8n8k4 f64 (SASS DMMA): the
// fp64 tensor path of sm_100a (tcgen05 has no f64 kind).
#pragma once
#include "common.cuh"

namespace fl {

struct WyArgs {
  const double* V;        // base of the V blocks
  const int64_t* voff;    // (J,) element offset of block j in V; nullptr: j * vstride
  int64_t vstride;
  const int32_t* vld;     // (J,) leading dimension; nullptr: vld_const
  int32_t vld_const;
  double* C;              // base of the C blocks
  const int64_t* coff;    // (J,) element offset of block j in C; nullptr: j * cstride
  int64_t cstride;
  const int32_t* cld;     // (J,); nullptr: cld_const
  int32_t cld_const;
  const int32_t* m;       // (J,) rows of block j
  const double* T;        // T_j at T + j * tstride, column-major NB x NB
  int64_t tstride;
  int64_t v_col0;         // first V column
  int64_t c_col0;         // first C column
  int32_t row0;           // first row; V's unit diagonal starts here
  int32_t transT;
  const int32_t* ncols;   // (J,) C columns of block j counted from column 0 of C...
  int32_t ncols_sub;      // ...minus ncols_sub (so tiles past a device-side rank exit)
  int32_t ncols_const;    // used when ncols == nullptr
  const int32_t* tiles;   // (ntiles, 2): block, first column (relative to c_col0); nullptr:
  int32_t tiles_per_block;//   block = blockIdx / tiles_per_block, column tile = remainder
  int32_t ntiles;
  const double* Csrc;     // null, or the store C is read from (same layout; written to C)
};

int wy_apply(const WyArgs& a, cudaStream_t s);               // NB = 32
int wy_apply_nb(const WyArgs& a, int nb, cudaStream_t s);    // NB = 32 or 64

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 256-bit global accesses (sm_100: LDG/STG.256): four consecutive doubles,
// 32-byte aligned. A warp access in the MMA fragment layout (8 columns x 4
// lanes) then covers one full 128-byte line per column instead of half.
struct d4 {
  double a, b, c, d;
};
__device__ __forceinline__ d4 ldg256(const double* p) {
  d4 v;
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n" : "=d"(v.a), "=d"(v.b), "=d"(v.c), "=d"(v.d) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg256(double* p, const d4& v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(v.a), "d"(v.b), "d"(v.c), "d"(v.d) : "memory");
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
// zero-fill form (src-size 0): the destination is written by the async unit,
// so it is ordered like the copies (used for out-of-range rows)
__device__ __forceinline__ void cp_async16_zero(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, 0;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// mbarrier helpers (shared::cta)
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(b)) : "memory");
}
// arrives on b when all of this thread's earlier cp.async copies have landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  unsigned done;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }\n"
                 : "=r"(done)
                 : "r"(smem_addr(b)), "r"(parity)
                 : "memory");
  } while (!done);
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace fl
