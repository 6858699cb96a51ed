// Device-side helpers shared by the libsem kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sem {
namespace dev {

// Programmatic dependent launch (PCG loop kernels): wait until the preceding
// grid has completed and its writes are visible, then let the next grid's CTAs
// be scheduled (they run their prologue and wait in turn).  Both are no-ops
// when the kernel was launched without the PDL attribute.
// Checked builds (build.py --variant checked -DSEM_CHECKED=1): the substitute
// for compute-sanitizer, which this pool does not allow.
// Every computed slot / buffer index of the gather-scatter, pack / unpack and
// exchange kernels is range-checked (and incidence slots must be ascending);
// a violation traps the kernel, so the next CUDA call fails loudly.  Device
// allocations are poisoned with 0xFF bytes (NaN doubles, -1 indices, 255
// multiplicities) so a read of never-written memory cannot go unnoticed.
#ifndef SEM_CHECKED
#define SEM_CHECKED 0
#endif
#define SEM_CHK(cond)                      \
  do {                                     \
    if (SEM_CHECKED && !(cond)) __trap();  \
  } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- PTX: mbarrier + bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA / bulk copy) accesses to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 16-byte global load / store with an L2 eviction-priority hint
__device__ __forceinline__ double2 ld2_hint(const double2* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st2_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
               "l"(pol)
               : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completion on mbarrier.
// dst, src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// atomic add with acquire-release semantics at GPU scope (returns old value)
__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------------------- reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed butterfly + serial over warps); blockDim a
// multiple of 32; result valid in thread 0.  `scratch` >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int q = 0; q < nw; q++) s += scratch[q];
  return s;
}

// Two-level deterministic grid reduction of NV values: every block writes its
// partials (partial[b*NV + q]); the last block to finish (atomic ticket)
// reduces them in a fixed order and writes out[q]; resets the ticket.
// Returns true in the last block (after out[] is written by thread 0).
template <int NV>
__device__ __forceinline__ bool grid_reduce(const double (&v)[NV], double* partial,
                                            unsigned* ticket, double* out, double* scratch,
                                            int* s_flag) {
  double bs[NV];
#pragma unroll
  for (int q = 0; q < NV; q++) bs[q] = block_sum(v[q], scratch);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; q++) partial[(size_t)blockIdx.x * NV + q] = bs[q];
    __threadfence();
    unsigned t = atomicAdd(ticket, 1u);
    *s_flag = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!*s_flag) return false;
  __threadfence();
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; q++) acc[q] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
#pragma unroll
    for (int q = 0; q < NV; q++) acc[q] += __ldcg(&partial[(size_t)b * NV + q]);
#pragma unroll
  for (int q = 0; q < NV; q++) {
    double s = block_sum(acc[q], scratch);
    if (threadIdx.x == 0) out[q] = s;
  }
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

// Geometric factors are stored element-blocked and plane-major,
// G[e][k][f][i + n j] with f in (rr, ss, tt, rs, rt, st): one k-plane of all six
// factors is a contiguous 48 n^2-byte block, the unit the Ax kernel streams.
__host__ __device__ __forceinline__ int64_t g_index(int64_t el, int f, int p, int n) {
  const int n2 = n * n, k = p / n2, ij = p - k * n2;
  return el * 6 * n2 * n + (int64_t)(k * 6 + f) * n2 + ij;
}

// ---------------------------------------------------------------- geometry
struct Box {
  double x0, x1, y0, y1, z0, z1;
};

// node coordinates (reading Q4)
__device__ __forceinline__ void node_xyz(const double* xi, int ex, int ey, int ez, int64_t e,
                                         int i, int j, int k, const Box& b, int deform,
                                         double amp, double* x) {
  const int64_t cx = e % ex, cy = (e / ex) % ey, cz = e / ((int64_t)ex * ey);
  const double hx = (b.x1 - b.x0) / ex, hy = (b.y1 - b.y0) / ey, hz = (b.z1 - b.z0) / ez;
  double X = b.x0 + hx * ((double)cx + 0.5 * (xi[i] + 1.0));
  double Y = b.y0 + hy * ((double)cy + 0.5 * (xi[j] + 1.0));
  double Z = b.z0 + hz * ((double)cz + 0.5 * (xi[k] + 1.0));
  if (deform) {
    const double tp = 6.283185307179586476925286766559;
    const double s = amp * sin(tp * (X - b.x0) / (b.x1 - b.x0)) *
                     sin(tp * (Y - b.y0) / (b.y1 - b.y0)) * sin(tp * (Z - b.z0) / (b.z1 - b.z0));
    X += s * (b.x1 - b.x0) / tp;
    Y += s * (b.y1 - b.y0) / tp;
    Z += s * (b.z1 - b.z0) / tp;
  }
  x[0] = X; x[1] = Y; x[2] = Z;
}

// slot-mask from the element's 6-bit Dirichlet face code (reading Q8)
__device__ __forceinline__ bool face_masked(unsigned bm, int i, int j, int k, int nm1) {
  return ((i == 0) && (bm & 1u)) || ((i == nm1) && (bm & 2u)) || ((j == 0) && (bm & 4u)) ||
         ((j == nm1) && (bm & 8u)) || ((k == 0) && (bm & 16u)) || ((k == nm1) && (bm & 32u));
}

}  // namespace dev
}  // namespace sem
