// ds_engine.cu -- device engine and C ABI for the sm_100a hot path of
// arXiv:1308.1536 (include/detseries_b200.h).
//
// Per pivot step i (elim.py:203-228; parexec.py:290-333 for the sharded form):
//   k_pivot   : exact zero test of the pivot (elim.py:209-212), pivots[i],
//               det chain det = piv | det*piv (elim.py:213-215)
//   k_mult    : z_j = RN(a_ji / piv) for this rank's rows j > i, a_ji <- -z_j
//               (elim.py:47, 53)
//   k_update  : a_jk <- RN(a_jk - RN(z_j * b_k)) for k != i (elim.py:49-52);
//               the real case runs the fused DFMA kernel of ds_update.cu
//   k_emit    : signed minors RN(det * L_{m,k}) + det, normalized RN(s_k/s_0)
//               for m = i+2 on the rank owning row i+1 (elim.py:56-61, 138-155)
// Kernels early-exit once the device abort flag holds a failed step, so the
// host never synchronises per step.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <string>
#include <algorithm>
#include <vector>

#include "ds_mp.cuh"
#include "ds_update.cuh"
#include "ds_tc.cuh"
#include "ds_warpdiv.cuh"
#include "ds_cwarp.cuh"

using namespace ds;

#define DS_VERSION "detseries_b200 0.1 (sm_100a)"

struct ds_ctx {
  int n, L, p, kind, ncomp, device, rank, world, nloc;
  // this context holds the rows row_base + rank + jl*world, jl < nloc: the
  // row-cyclic shard of a rank (row_base 0), or a block of consecutive rows
  // (world 1) of the panel-paged executor (ds_create_block)
  int row_base;
  cudaStream_t stream, own_stream;
  cudaStream_t side;           // det chain + minors emission (outputs only, may lag)
  cudaEvent_t ev, ev_piv, ev_upd;
  double *ws_dx, *ws_dy, *ws_ex, *ws_ey;  // side-stream product workspaces
  // matrix rows owned by this rank: [ncomp][L][nloc*n] limbs
  uint32_t* a_limbs;
  int32_t* a_exp;
  uint8_t* a_cls;
  int64_t a_count;
  // broadcast pivot buffer (same byte layout as the oracle's)
  uint8_t* pbuf;       // active pivot buffer (own or caller-provided)
  uint8_t* own_pbuf;
  size_t pbuf_bytes;
  // multipliers z_j for local rows: [ncomp][L][nloc]
  uint32_t* z_limbs;   // multipliers of the current step (= zb_*[step & 1])
  int32_t* z_exp;
  uint8_t* z_cls;
  uint32_t* zb_limbs[2];  // double buffer: the lookahead writes step i+1's multipliers
  int32_t* zb_exp[2];     // while step i's update still reads step i's
  uint8_t* zb_cls[2];
  // lookahead (world 1, tensor-core update): the column tile holding column
  // i+1 is updated first on `la`, then step i+1's multipliers are computed
  // there while the rest of step i's update runs on the main stream
  cudaStream_t la;
  cudaEvent_t ev_prep, ev_a, ev_mult, ev_la_done;
  int la_step;   // the step whose multipliers are already computed (-1: none)
  int la_limit;  // lookahead only for steps i + 1 < la_limit (set by ds_run / ds_lookahead_enable)
  int la_ext;    // multi-rank: the caller exchanges the next pivot (ds_lookahead_pivot / _mult)
  // trace: pivots/dets [ncomp][L][n]; det running value [ncomp][L][1]
  uint32_t *piv_limbs, *det_limbs, *cur_limbs;
  int32_t *piv_exp, *det_exp, *cur_exp;
  uint8_t *piv_cls, *det_cls, *cur_cls;
  // minors for owned rows: [ncomp][L][nloc*n] (row m-1 local index (m-1)/world)
  uint32_t *sig_limbs, *nrm_limbs;
  int32_t *sig_exp, *nrm_exp;
  uint8_t *sig_cls, *nrm_cls;
  uint8_t* row_flags;  // [n]
  // minors storage: m_rows local rows (all nloc, or a ring while streaming), plane stride m_count
  int m_rows;
  int64_t m_count;
  // streaming of minors rows to the host (ds_stream_minors / ds_stream_flush)
  int st_batch;              // max steps between flushes (ring sized for it); 0 = off
  ds_rows_cb st_cb;
  void* st_user;
  int st_next;               // first global row not yet copied
  int st_set;                // staging set of the copy in flight
  int st_pending;            // a copy is in flight in set st_set
  int st_pend_g0, st_pend_rows, st_pend_width;
  int st_rows_cap;           // rows per staging set
  uint32_t* st_limbs[2][2];  // [set][signed / normalized] pinned host staging
  int32_t* st_exp[2][2];
  uint8_t* st_cls[2][2];
  uint8_t* st_flags[2];
  cudaEvent_t st_ev[2];
  // status: [0] failed step (-1), [1] have_det, [2] range error count, [3] warnings
  int32_t* status;
  // per-thread scratch for the general engine
  uint32_t* scratch;
  int64_t scratch_threads;
  int64_t scratch_words;  // words per thread
  uint32_t* scratch_side; // complex tensor-core runs: general kernels on the side stream (det chain, minors)
  // device snapshot of the local rows (ds_snapshot)
  uint32_t* snap_limbs;
  int32_t* snap_exp;
  uint8_t* snap_cls;
  // update profiling
  int prof_on;
  std::vector<cudaEvent_t> prof_ev;  // pairs
  size_t prof_used;
  int64_t prof_launches;
  double prof_work;
  // fused update engine workspace
  UpdatePlan plan;
  TcPlan tc;  // tensor-core update (tcgen05 kind::i8), preferred when enabled
  int64_t launches;
  int64_t h2d_bytes, d2h_bytes;  // host<->device bytes moved by the ABI copies (e2e accounting)
  int host_have_det;   // a det chain value exists (first step sets det = piv)
  int det_from_cur;    // next det product reads the ds_set_det seed in `cur`
  // pivot_mode="partial" (elim.py:204-208): per-step row swap flags [n] and the selected row
  int pivot_partial;
  uint8_t* swaps;
  int32_t* pbest;
  std::string err;
};

static std::string g_last_error;

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      if (ctx) ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);      \
      g_last_error = std::string(#call) + ": " + cudaGetErrorString(e_);           \
      return DS_CUDA;                                                              \
    }                                                                              \
  } while (0)

static inline int nlimbs(long p) { return (int)((p + 31) / 32); }

static size_t pbuf_size(int n, int L, int ncomp) {
  return (size_t)4 * ncomp * L * n + (size_t)4 * ncomp * n + (((size_t)ncomp * n + 3) & ~(size_t)3);
}

struct PB {  // pivot buffer view
  uint32_t* limbs;
  int32_t* exp;
  uint8_t* cls;
};
__host__ __device__ static inline PB pb_view(uint8_t* p, int n, int L, int ncomp) {
  PB v;
  v.limbs = (uint32_t*)p;
  v.exp = (int32_t*)(p + (size_t)4 * ncomp * L * n);
  v.cls = (uint8_t*)(p + (size_t)4 * ncomp * L * n + (size_t)4 * ncomp * n);
  return v;
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ Val val_at(const uint32_t* limbs, const int32_t* ex, const uint8_t* cl, int64_t count,
                                      int c, int L, int64_t idx) {
  Val v;
  v.m = CPtr{limbs + (int64_t)c * L * count + idx, count};
  v.e = ex[(int64_t)c * count + idx];
  v.c = cl[(int64_t)c * count + idx];
  return v;
}

struct Out {
  Ptr m;
  int32_t* e;
  uint8_t* c;
};
__device__ __forceinline__ Out out_at(uint32_t* limbs, int32_t* ex, uint8_t* cl, int64_t count, int c, int L,
                                      int64_t idx) {
  Out o;
  o.m = Ptr{limbs + (int64_t)c * L * count + idx, count};
  o.e = ex + (int64_t)c * count + idx;
  o.c = cl + (int64_t)c * count + idx;
  return o;
}

__device__ __forceinline__ void neg_copy(Out o, const Val& v, int L) {
  for (int l = 0; l < L; l++) o.m[l] = v.m[l];
  *o.e = (int32_t)v.e;
  uint8_t c = v.c;
  *o.c = (c == DS_CLS_POS) ? DS_CLS_NEG : (c == DS_CLS_NEG) ? DS_CLS_POS : (c == DS_CLS_PZERO) ? DS_CLS_NZERO : DS_CLS_PZERO;
}

__device__ __forceinline__ void set_val(Out o, const Val& v, int L) {
  for (int l = 0; l < L; l++) o.m[l] = v.m[l];
  *o.e = (int32_t)v.e;
  *o.c = v.c;
}

// generic scalar ops on one (possibly complex) value; scratch tmp per thread
__device__ bool g_mul(Out o0, Out o1, Val a0, Val a1, Val b0, Val b1, int kind, int L, int p, Ptr tmp) {
  if (kind == DS_KIND_REAL) return mul_rn(o0.m, o0.e, o0.c, a0, b0, L, p, tmp);
  bool ok = cmul_part(o0.m, o0.e, o0.c, a0, b0, a1, b1, true, L, p, tmp);
  ok &= cmul_part(o1.m, o1.e, o1.c, a0, b1, a1, b0, false, L, p, tmp);
  return ok;
}

__device__ bool g_div(Out o0, Out o1, Val a0, Val a1, Val b0, Val b1, int kind, int L, int p, Ptr tmp,
                      unsigned int* warn) {
  if (kind == DS_KIND_REAL) return div_rn(o0.m, o0.e, o0.c, a0, b0, L, p, tmp);
  bool ok = cdiv_part(o0.m, o0.e, o0.c, a0, a1, b0, b1, false, L, p, tmp, warn);
  ok &= cdiv_part(o1.m, o1.e, o1.c, a0, a1, b0, b1, true, L, p, tmp, warn);
  return ok;
}

__device__ bool g_sub(Out o0, Out o1, Val a0, Val a1, Val b0, Val b1, int kind, int L, int p, Ptr tmp) {
  bool ok = add_rn(o0.m, o0.e, o0.c, a0, b0, true, L, p, tmp);
  if (kind == DS_KIND_COMPLEX) ok &= add_rn(o1.m, o1.e, o1.c, a1, b1, true, L, p, tmp);
  return ok;
}

__device__ bool g_add(Out o0, Out o1, Val a0, Val a1, Val b0, Val b1, int kind, int L, int p, Ptr tmp) {
  bool ok = add_rn(o0.m, o0.e, o0.c, a0, b0, false, L, p, tmp);
  if (kind == DS_KIND_COMPLEX) ok &= add_rn(o1.m, o1.e, o1.c, a1, b1, false, L, p, tmp);
  return ok;
}

// ---------------------------------------------------------------- kernels
struct KArgs {
  int n, L, p, kind, ncomp, rank, world, nloc, row_base;
  uint32_t* a_limbs; int32_t* a_exp; uint8_t* a_cls; int64_t a_count;
  uint8_t* pbuf;
  uint32_t* z_limbs; int32_t* z_exp; uint8_t* z_cls;
  uint32_t *piv_limbs, *det_limbs, *cur_limbs;
  int32_t *piv_exp, *det_exp, *cur_exp;
  uint8_t *piv_cls, *det_cls, *cur_cls;
  uint32_t *sig_limbs, *nrm_limbs;
  int32_t *sig_exp, *nrm_exp;
  uint8_t *sig_cls, *nrm_cls;
  uint8_t* row_flags;
  int32_t* status;
  uint32_t* scratch; int64_t scratch_threads; int64_t scratch_words;
  int64_t m_count; int m_rows;  // minors storage: plane stride, ring rows (local row jl -> slot jl % m_rows)
  int sm_threads;  // > 0: the thread-level kernel keeps its scratch in shared memory (blockDim threads)
};

static KArgs kargs(ds_ctx* c) {
  KArgs k;
  k.n = c->n; k.L = c->L; k.p = c->p; k.kind = c->kind; k.ncomp = c->ncomp; k.rank = c->rank;
  k.world = c->world; k.nloc = c->nloc; k.row_base = c->row_base;
  k.a_limbs = c->a_limbs; k.a_exp = c->a_exp; k.a_cls = c->a_cls; k.a_count = c->a_count;
  k.pbuf = c->pbuf;
  k.z_limbs = c->z_limbs; k.z_exp = c->z_exp; k.z_cls = c->z_cls;
  k.piv_limbs = c->piv_limbs; k.det_limbs = c->det_limbs; k.cur_limbs = c->cur_limbs;
  k.piv_exp = c->piv_exp; k.det_exp = c->det_exp; k.cur_exp = c->cur_exp;
  k.piv_cls = c->piv_cls; k.det_cls = c->det_cls; k.cur_cls = c->cur_cls;
  k.sig_limbs = c->sig_limbs; k.nrm_limbs = c->nrm_limbs; k.sig_exp = c->sig_exp; k.nrm_exp = c->nrm_exp;
  k.sig_cls = c->sig_cls; k.nrm_cls = c->nrm_cls; k.row_flags = c->row_flags; k.status = c->status;
  k.scratch = c->scratch; k.scratch_threads = c->scratch_threads; k.scratch_words = c->scratch_words;
  k.m_count = c->m_count; k.m_rows = c->m_rows;
  k.sm_threads = 0;
  return k;
}

// per-thread scratch of the thread-level (complex) kernels: shared memory when
// the launch gave each thread its words there (latency ~30 cycles instead of an
// L2 round trip per limb in the O(L^2) exact products and divisions), else global
__device__ __forceinline__ Ptr kscratch(const KArgs& k, int64_t tid) {
  if (k.sm_threads) {
    extern __shared__ uint32_t ksm[];
    return Ptr{ksm + threadIdx.x, (int64_t)blockDim.x};
  }
  return Ptr{k.scratch + tid, k.scratch_threads};
}

// operand q (0..3) of this thread copied into shared memory after its scratch
// (the O(L^2) product loops re-read every operand limb L times: from global
// memory each limb is a separate line, and the large shared-memory carve-out
// leaves little L1 to hold them)
__device__ __forceinline__ Val kstage(const KArgs& k, const Val& v, int q) {
  if (!k.sm_threads) return v;
  extern __shared__ uint32_t ksm[];
  const int64_t T = blockDim.x;
  uint32_t* dst = ksm + (k.scratch_words + (int64_t)q * k.L) * T + threadIdx.x;
  for (int l = 0; l < k.L; l++) dst[(int64_t)l * T] = v.m[l];
  Val o;
  o.m = CPtr{dst, T};
  o.e = v.e;
  o.c = v.c;
  return o;
}

// first element of local row jl's minors slot (ring of m_rows rows)
__device__ __forceinline__ int64_t mrow(const KArgs& k, int64_t jl) { return (jl % k.m_rows) * k.n; }

__device__ __forceinline__ Ptr thread_scratch(const KArgs& k, int64_t tid) {
  return Ptr{k.scratch + tid, k.scratch_threads};
}

// owner stages its row i into the pivot buffer: one thread per (component,
// limb plane, column), coalesced along the row
__global__ void k_stage(KArgs k, int i) {
  if (k.status[0] >= 0) return;
  int64_t jl = (i - k.row_base) / k.world;
  PB pb = pb_view(k.pbuf, k.n, k.L, k.ncomp);
  int64_t planes = (int64_t)k.ncomp * (k.L + 2);  // L limb planes + exp + cls per component
  int64_t tot = planes * k.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    int col = (int)(t % k.n);
    int64_t pl = t / k.n;
    int c = (int)(pl / (k.L + 2));
    int l = (int)(pl % (k.L + 2));
    int64_t src = jl * k.n + col;
    if (l < k.L)
      pb.limbs[((int64_t)c * k.L + l) * k.n + col] = k.a_limbs[((int64_t)c * k.L + l) * k.a_count + src];
    else if (l == k.L)
      pb.exp[(int64_t)c * k.n + col] = k.a_exp[(int64_t)c * k.a_count + src];
    else
      pb.cls[(int64_t)c * k.n + col] = k.a_cls[(int64_t)c * k.a_count + src];
  }
}

// ---- pivot_mode="partial" (elim.py:204-208, det-only; world 1, real) ----
// |a_x| < |a_y| for two real matrix elements (abs() comparison of elim.py:205,
// exact): zeros are the smallest magnitude, then exponent, then the mantissa
// limbs from the most significant (limb L-1) down
__device__ __forceinline__ bool abs_less(const KArgs& k, int64_t ix, int64_t iy) {
  if (is_zero_cls(k.a_cls[iy])) return false;
  if (is_zero_cls(k.a_cls[ix])) return true;
  int32_t ex = k.a_exp[ix], ey = k.a_exp[iy];
  if (ex != ey) return ex < ey;
  for (int l = k.L - 1; l >= 0; l--) {
    uint32_t x = k.a_limbs[(int64_t)l * k.a_count + ix], y = k.a_limbs[(int64_t)l * k.a_count + iy];
    if (x != y) return x < y;
  }
  return false;
}

// best = the first row j >= i of maximal |a_ji| (Python max() keeps the first
// maximum); one block, strided scan then a tree reduction with index tie-break
__global__ void k_pivot_select(KArgs k, int i, int32_t* best, uint8_t* swaps) {
  __shared__ int cand[1024];
  const int t = threadIdx.x;
  if (k.status[0] >= 0) {  // an earlier step aborted: nothing moves
    if (t == 0) { *best = i; swaps[i] = 0; }
    return;
  }
  int b = -1;
  for (int j = i + t; j < k.n; j += blockDim.x)
    if (b < 0 || abs_less(k, (int64_t)b * k.n + i, (int64_t)j * k.n + i)) b = j;
  cand[t] = b;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (t < h) {
      int x = cand[t], y = cand[t + h];
      if (y >= 0) {
        bool take = x < 0;
        if (!take) {
          int64_t ix = (int64_t)x * k.n + i, iy = (int64_t)y * k.n + i;
          take = abs_less(k, ix, iy) || (y < x && !abs_less(k, iy, ix));
        }
        if (take) cand[t] = y;
      }
    }
    __syncthreads();
  }
  if (t == 0) {
    int bb = cand[0] < 0 ? i : cand[0];
    *best = bb;
    swaps[i] = bb != i;
  }
}

// rows[i], rows[best] = rows[best], rows[i] (elim.py:206-207): every limb plane,
// exponent and class of both full-width rows, coalesced along the rows
__global__ void k_swap_rows(KArgs k, int i, const int32_t* best) {
  const int b = *best;
  if (b == i) return;
  const int64_t planes = (int64_t)k.ncomp * (k.L + 2);
  const int64_t tot = planes * k.n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int col = (int)(t % k.n);
    const int64_t pl = t / k.n;
    const int c = (int)(pl / (k.L + 2));
    const int l = (int)(pl % (k.L + 2));
    const int64_t x = (int64_t)i * k.n + col, y = (int64_t)b * k.n + col;
    if (l < k.L) {
      uint32_t* a = k.a_limbs + ((int64_t)c * k.L + l) * k.a_count;
      uint32_t u = a[x]; a[x] = a[y]; a[y] = u;
    } else if (l == k.L) {
      int32_t* a = k.a_exp + (int64_t)c * k.a_count;
      int32_t u = a[x]; a[x] = a[y]; a[y] = u;
    } else {
      uint8_t* a = k.a_cls + (int64_t)c * k.a_count;
      uint8_t u = a[x]; a[x] = a[y]; a[y] = u;
    }
  }
}

// zero test + pivots[i] + det chain (single thread, general engine)
__global__ void k_pivot(KArgs k, int i) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (k.status[0] >= 0) return;
  PB pb = pb_view(k.pbuf, k.n, k.L, k.ncomp);
  Val p0 = val_at(pb.limbs, pb.exp, pb.cls, k.n, 0, k.L, i);
  Val p1 = k.kind == DS_KIND_COMPLEX ? val_at(pb.limbs, pb.exp, pb.cls, k.n, 1, k.L, i) : p0;
  bool zero = is_zero_cls(p0.c) && (k.kind == DS_KIND_REAL || is_zero_cls(p1.c));
  if (zero) {  // elim.py:209-212 exact zero only
    k.status[0] = i;
    return;
  }
  Out pv0 = out_at(k.piv_limbs, k.piv_exp, k.piv_cls, k.n, 0, k.L, i);
  Out pv1 = out_at(k.piv_limbs, k.piv_exp, k.piv_cls, k.n, k.ncomp - 1, k.L, i);
  set_val(pv0, p0, k.L);
  if (k.kind == DS_KIND_COMPLEX) set_val(pv1, p1, k.L);
  Out c0 = out_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, 0, k.L, 0);
  Out c1 = out_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, k.ncomp - 1, k.L, 0);
  Out d0 = out_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 0, k.L, i);
  Out d1 = out_at(k.det_limbs, k.det_exp, k.det_cls, k.n, k.ncomp - 1, k.L, i);
  if (!k.status[1]) {  // det = piv (unrounded, elim.py:214)
    set_val(c0, p0, k.L);
    if (k.kind == DS_KIND_COMPLEX) set_val(c1, p1, k.L);
    k.status[1] = 1;
  } else {
    // det*piv into d (scratch), then copy to cur
    Val q0 = val_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, 0, k.L, 0);
    Val q1 = val_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, k.ncomp - 1, k.L, 0);
    Ptr tmp = thread_scratch(k, 0);
    if (!g_mul(d0, d1, q0, q1, p0, p1, k.kind, k.L, k.p, tmp)) atomicAdd(&k.status[2], 1);
    Val r0 = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 0, k.L, i);
    Val r1 = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, k.ncomp - 1, k.L, i);
    set_val(c0, r0, k.L);
    if (k.kind == DS_KIND_COMPLEX) set_val(c1, r1, k.L);
    return;
  }
  Val r0 = val_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, 0, k.L, 0);
  Val r1 = val_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, k.ncomp - 1, k.L, 0);
  set_val(d0, r0, k.L);
  if (k.kind == DS_KIND_COMPLEX) set_val(d1, r1, k.L);
}

// det_i = RN(det_{i-1} * piv_i) (elim.py:215) by one thread, on the side stream
// (complex tensor-core runs); from_cur: the ds_set_det seed in cur is det_{i-1}
__global__ void k_det_step(KArgs k, int i, int from_cur) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (k.status[0] >= 0 && k.status[0] <= i) return;
  Val q0 = from_cur ? val_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, 0, k.L, 0)
                    : val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 0, k.L, i - 1);
  Val q1 = from_cur ? val_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, k.ncomp - 1, k.L, 0)
                    : val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, k.ncomp - 1, k.L, i - 1);
  Val p0 = val_at(k.piv_limbs, k.piv_exp, k.piv_cls, k.n, 0, k.L, i);
  Val p1 = val_at(k.piv_limbs, k.piv_exp, k.piv_cls, k.n, k.ncomp - 1, k.L, i);
  Out d0 = out_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 0, k.L, i);
  Out d1 = out_at(k.det_limbs, k.det_exp, k.det_cls, k.n, k.ncomp - 1, k.L, i);
  q0 = kstage(k, q0, 0);
  q1 = kstage(k, q1, 1);
  p0 = kstage(k, p0, 2);
  p1 = kstage(k, p1, 3);
  if (!g_mul(d0, d1, q0, q1, p0, p1, k.kind, k.L, k.p, kscratch(k, 0))) atomicAdd(&k.status[2], 1);
}

// first local row index with global row > i (global = row_base + rank + jl*world)
__host__ __device__ static inline int first_local_after(int i, int rank, int world, int row_base = 0) {
  int first = i + 1 - row_base;
  if (first <= rank) return 0;
  return (first - rank + world - 1) / world;
}

// does this context hold global row g
static inline bool owns_row(const ds_ctx* c, int g) {
  const int r = g - c->row_base;
  return r >= 0 && r % c->world == c->rank && r / c->world < c->nloc;
}

// z_j = RN(a_ji / piv), a_ji <- -z_j  (elim.py:47, 53)
__global__ void k_mult(KArgs k, int i, int jl0) {
  if (k.status[0] >= 0) return;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int nrows = k.nloc - jl0;
  PB pb = pb_view(k.pbuf, k.n, k.L, k.ncomp);
  Val b0 = val_at(pb.limbs, pb.exp, pb.cls, k.n, 0, k.L, i);
  Val b1 = k.kind == DS_KIND_COMPLEX ? val_at(pb.limbs, pb.exp, pb.cls, k.n, 1, k.L, i) : b0;
  for (int64_t r = tid; r < nrows; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t jl = jl0 + r;
    int64_t idx = jl * k.n + i;
    Val a0 = val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, idx);
    Val a1 = k.kind == DS_KIND_COMPLEX ? val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 1, k.L, idx) : a0;
    Out z0 = out_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, 0, k.L, jl);
    Out z1 = out_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, k.ncomp - 1, k.L, jl);
    Ptr tmp = thread_scratch(k, tid);
    if (!g_div(z0, z1, a0, a1, b0, b1, k.kind, k.L, k.p, tmp, (unsigned int*)&k.status[3]))
      atomicAdd(&k.status[2], 1);
    Val zv0 = val_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, 0, k.L, jl);
    Out ao0 = out_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, idx);
    neg_copy(ao0, zv0, k.L);
    if (k.kind == DS_KIND_COMPLEX) {
      Val zv1 = val_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, 1, k.L, jl);
      Out ao1 = out_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 1, k.L, idx);
      neg_copy(ao1, zv1, k.L);
    }
  }
}

// complex (tensor-core runs): one thread per (row, component) for the division,
// twice the parallelism of k_mult; a_ji <- -z_j after all rows (k_neg_z), since
// both components of a_ji are read by both threads
__global__ void k_mult_c2(KArgs k, int i, int jl0) {
  if (k.status[0] >= 0) return;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int nrows = k.nloc - jl0;
  PB pb = pb_view(k.pbuf, k.n, k.L, k.ncomp);
  Val b0 = val_at(pb.limbs, pb.exp, pb.cls, k.n, 0, k.L, i);
  Val b1 = val_at(pb.limbs, pb.exp, pb.cls, k.n, 1, k.L, i);
  for (int64_t t = tid; t < 2 * (int64_t)nrows; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t & 1);
    int64_t jl = jl0 + (t >> 1);
    int64_t idx = jl * k.n + i;
    Val a0 = kstage(k, val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, idx), 0);
    Val a1 = kstage(k, val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 1, k.L, idx), 1);
    Out z = out_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, c, k.L, jl);
    if (!cdiv_part(z.m, z.e, z.c, a0, a1, kstage(k, b0, 2), kstage(k, b1, 3), c == 1, k.L, k.p, kscratch(k, tid),
                   (unsigned int*)&k.status[3]))
      atomicAdd(&k.status[2], 1);
  }
}

__global__ void k_neg_z(KArgs k, int i, int jl0) {
  if (k.status[0] >= 0) return;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int nrows = k.nloc - jl0;
  for (int64_t t = tid; t < 2 * (int64_t)nrows; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t & 1);
    int64_t jl = jl0 + (t >> 1);
    Val zv = val_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, c, k.L, jl);
    neg_copy(out_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, c, k.L, jl * k.n + i), zv, k.L);
  }
}

// complex minors, one thread per (entry, component): signed_k = RN(det_i * L_mk)
// (cmul_part per component), normalized = RN(signed_k / signed_0) (cdiv_part)
__global__ void k_emit_signed_c2(KArgs k, int i) {
  // side stream: a zero pivot found by a LATER step must not cancel this row (elim.py:220-226
  // emits size i+2 before step i+1 raises)
  if (k.status[0] >= 0 && k.status[0] <= i) return;
  int m = i + 2;
  int64_t jl = (i + 1 - k.row_base) / k.world;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  Val d0 = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 0, k.L, i);
  Val d1 = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 1, k.L, i);
  for (int64_t t = tid; t < 2 * (int64_t)m; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t & 1);
    const int64_t kk = t >> 1;
    int64_t oidx = jl * k.n + kk;
    Out so = out_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, c, k.L, mrow(k, jl) + kk);
    if (kk == m - 1) {
      set_val(so, c == 0 ? d0 : d1, k.L);
      continue;
    }
    const Val a0 = kstage(k, val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, oidx), 0);
    const Val a1 = kstage(k, val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 1, k.L, oidx), 1);
    const Val e0 = kstage(k, d0, 2), e1 = kstage(k, d1, 3);
    bool ok = c == 0 ? cmul_part(so.m, so.e, so.c, e0, a0, e1, a1, true, k.L, k.p, kscratch(k, tid))
                     : cmul_part(so.m, so.e, so.c, e0, a1, e1, a0, false, k.L, k.p, kscratch(k, tid));
    if (!ok) atomicAdd(&k.status[2], 1);
  }
}

__global__ void k_emit_norm_c2(KArgs k, int i) {
  if (k.status[0] >= 0 && k.status[0] <= i) return;  // see k_emit_signed_c2
  int m = i + 2;
  int64_t jl = (i + 1 - k.row_base) / k.world;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r0 = mrow(k, jl);
  Val l0 = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, r0);
  Val l1 = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 1, k.L, r0);
  bool lead_zero = is_zero_cls(l0.c) && is_zero_cls(l1.c);
  if (tid == 0) k.row_flags[m - 1] = lead_zero ? 1 : 3;
  if (lead_zero) return;
  for (int64_t t = tid; t < 2 * (int64_t)m; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t & 1);
    int64_t idx = r0 + (t >> 1);
    const Val s0 = kstage(k, val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, idx), 0);
    const Val s1 = kstage(k, val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 1, k.L, idx), 1);
    Out o = out_at(k.nrm_limbs, k.nrm_exp, k.nrm_cls, k.m_count, c, k.L, idx);
    if (!cdiv_part(o.m, o.e, o.c, s0, s1, kstage(k, l0, 2), kstage(k, l1, 3), c == 1, k.L, k.p, kscratch(k, tid),
                   (unsigned int*)&k.status[3]))
      atomicAdd(&k.status[2], 1);
  }
}

// ---- complex step on warps (ds_cwarp.cuh): one warp per (item, component),
// each warp with its own shared-memory region of cw_words words
__device__ __forceinline__ dscw::Region cw_region(const KArgs& k, int cw_words) {
  extern __shared__ uint32_t cwsm[];
  return dscw::Region(cwsm + (int64_t)(threadIdx.x >> 5) * cw_words, k.L, k.p);
}

// z_j = RN(a_ji / piv) per component (elim.py:47); a_ji <- -z_j by k_neg_z
__global__ void k_cw_mult(KArgs k, int i, int jl0, int cw_words) {
  if (k.status[0] >= 0) return;
  const int wpb = blockDim.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  const int nrows = k.nloc - jl0;
  if (t >= 2 * (int64_t)nrows) return;
  dscw::Region R = cw_region(k, cw_words);
  const int c = (int)(t & 1);
  const int64_t jl = jl0 + (t >> 1);
  const int64_t idx = jl * k.n + i;
  PB pb = pb_view(k.pbuf, k.n, k.L, k.ncomp);
  const Val a0 = dscw::stage(val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, idx), R.op, k.L);
  const Val a1 = dscw::stage(val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 1, k.L, idx), R.op + k.L, k.L);
  const Val b0 = dscw::stage(val_at(pb.limbs, pb.exp, pb.cls, k.n, 0, k.L, i), R.op + 2 * k.L, k.L);
  const Val b1 = dscw::stage(val_at(pb.limbs, pb.exp, pb.cls, k.n, 1, k.L, i), R.op + 3 * k.L, k.L);
  __syncwarp();
  Out z = out_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, c, k.L, jl);
  if (!dscw::wcdiv_part(z.m, z.e, z.c, a0, a1, b0, b1, c == 1, k.L, k.p, R, (unsigned int*)&k.status[3]) &&
      (threadIdx.x & 31) == 0)
    atomicAdd(&k.status[2], 1);
}

// det_i = RN(det_{i-1} * piv_i) per component (elim.py:213-215); 2 warps
__global__ void k_cw_det(KArgs k, int i, int from_cur, int cw_words) {
  if (k.status[0] >= 0 && k.status[0] <= i) return;
  const int c = threadIdx.x >> 5;
  if (c > 1) return;
  dscw::Region R = cw_region(k, cw_words);
  const Val q0 = dscw::stage(from_cur ? val_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, 0, k.L, 0)
                                      : val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 0, k.L, i - 1),
                             R.op, k.L);
  const Val q1 = dscw::stage(from_cur ? val_at(k.cur_limbs, k.cur_exp, k.cur_cls, 1, 1, k.L, 0)
                                      : val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 1, k.L, i - 1),
                             R.op + k.L, k.L);
  const Val p0 = dscw::stage(val_at(k.piv_limbs, k.piv_exp, k.piv_cls, k.n, 0, k.L, i), R.op + 2 * k.L, k.L);
  const Val p1 = dscw::stage(val_at(k.piv_limbs, k.piv_exp, k.piv_cls, k.n, 1, k.L, i), R.op + 3 * k.L, k.L);
  __syncwarp();
  Out d = out_at(k.det_limbs, k.det_exp, k.det_cls, k.n, c, k.L, i);
  // re = q0 p0 - q1 p1, im = q0 p1 + q1 p0 (g_mul / cmul_part order)
  const bool ok = c == 0 ? dscw::wcmul_part(d.m, d.e, d.c, q0, p0, q1, p1, true, k.L, k.p, R)
                         : dscw::wcmul_part(d.m, d.e, d.c, q0, p1, q1, p0, false, k.L, k.p, R);
  if (!ok && (threadIdx.x & 31) == 0) atomicAdd(&k.status[2], 1);
}

// signed minors of size m = i+2 per component (elim.py:56-61)
__global__ void k_cw_emit_signed(KArgs k, int i, int cw_words) {
  if (k.status[0] >= 0 && k.status[0] <= i) return;  // see k_emit_signed_c2
  const int m = i + 2;
  const int64_t jl = (i + 1 - k.row_base) / k.world;
  const int wpb = blockDim.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  if (t >= 2 * (int64_t)m) return;
  const int c = (int)(t & 1);
  const int64_t kk = t >> 1;
  Out so = out_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, c, k.L, mrow(k, jl) + kk);
  const Val d0r = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 0, k.L, i);
  const Val d1r = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 1, k.L, i);
  if (kk == m - 1) {
    const Val& dv = c == 0 ? d0r : d1r;
    for (int l = threadIdx.x & 31; l < k.L; l += 32) so.m[l] = dv.m[l];
    if ((threadIdx.x & 31) == 0) {
      *so.e = (int32_t)dv.e;
      *so.c = dv.c;
    }
    return;
  }
  dscw::Region R = cw_region(k, cw_words);
  const int64_t oidx = jl * k.n + kk;
  const Val a0 = dscw::stage(val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, oidx), R.op, k.L);
  const Val a1 = dscw::stage(val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 1, k.L, oidx), R.op + k.L, k.L);
  const Val d0 = dscw::stage(d0r, R.op + 2 * k.L, k.L);
  const Val d1 = dscw::stage(d1r, R.op + 3 * k.L, k.L);
  __syncwarp();
  const bool ok = c == 0 ? dscw::wcmul_part(so.m, so.e, so.c, d0, a0, d1, a1, true, k.L, k.p, R)
                         : dscw::wcmul_part(so.m, so.e, so.c, d0, a1, d1, a0, false, k.L, k.p, R);
  if (!ok && (threadIdx.x & 31) == 0) atomicAdd(&k.status[2], 1);
}

// normalized minors RN(s_k / s_0) per component (elim.py:138-155)
__global__ void k_cw_emit_norm(KArgs k, int i, int cw_words) {
  if (k.status[0] >= 0 && k.status[0] <= i) return;
  const int m = i + 2;
  const int64_t jl = (i + 1 - k.row_base) / k.world;
  const int64_t r0 = mrow(k, jl);
  const Val l0r = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, r0);
  const Val l1r = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 1, k.L, r0);
  const bool lead_zero = is_zero_cls(l0r.c) && is_zero_cls(l1r.c);
  if (blockIdx.x == 0 && threadIdx.x == 0) k.row_flags[m - 1] = lead_zero ? 1 : 3;
  if (lead_zero) return;
  const int wpb = blockDim.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5);
  if (t >= 2 * (int64_t)m) return;
  const int c = (int)(t & 1);
  const int64_t idx = r0 + (t >> 1);
  dscw::Region R = cw_region(k, cw_words);
  const Val s0 = dscw::stage(val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, idx), R.op, k.L);
  const Val s1 = dscw::stage(val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 1, k.L, idx), R.op + k.L, k.L);
  const Val l0 = dscw::stage(l0r, R.op + 2 * k.L, k.L);
  const Val l1 = dscw::stage(l1r, R.op + 3 * k.L, k.L);
  __syncwarp();
  Out o = out_at(k.nrm_limbs, k.nrm_exp, k.nrm_cls, k.m_count, c, k.L, idx);
  if (!dscw::wcdiv_part(o.m, o.e, o.c, s0, s1, l0, l1, c == 1, k.L, k.p, R, (unsigned int*)&k.status[3]) &&
      (threadIdx.x & 31) == 0)
    atomicAdd(&k.status[2], 1);
}

// general-engine update: a_jk <- RN(a_jk - RN(z_j * b_k)); used for complex
// values (4 exact products per element) and as the reference path the fused
// real kernel is tested against.
__global__ void k_update_general(KArgs k, int i, int jl0, int collect_minors) {
  if (k.status[0] >= 0) return;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int nrows = k.nloc - jl0;
  int kfirst = collect_minors ? 0 : i + 1;
  int ncols = k.n - kfirst - (collect_minors ? 1 : 0);  // all k != i in range
  if (ncols <= 0) return;
  int64_t total = (int64_t)nrows * ncols;
  PB pb = pb_view(k.pbuf, k.n, k.L, k.ncomp);
  Ptr tmp = thread_scratch(k, tid);
  Ptr tv = tmp;                  // t components: 2 * L limbs
  Ptr work = tmp.off(2 * (int64_t)k.L + 4);
  int32_t te[2];
  uint8_t tc[2];
  for (int64_t w = tid; w < total; w += (int64_t)gridDim.x * blockDim.x) {
    int64_t jl = jl0 + w / ncols;
    int kk = kfirst + (int)(w % ncols);
    if (collect_minors && kk >= i) kk += 1;  // skip column i
    int64_t idx = jl * k.n + kk;
    Val z0 = val_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, 0, k.L, jl);
    Val z1 = k.kind == DS_KIND_COMPLEX ? val_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, 1, k.L, jl) : z0;
    Val b0 = val_at(pb.limbs, pb.exp, pb.cls, k.n, 0, k.L, kk);
    Val b1 = k.kind == DS_KIND_COMPLEX ? val_at(pb.limbs, pb.exp, pb.cls, k.n, 1, k.L, kk) : b0;
    Out t0{tv, &te[0], &tc[0]};
    Out t1{tv.off(k.L), &te[1], &tc[1]};
    bool ok = g_mul(t0, t1, z0, z1, b0, b1, k.kind, k.L, k.p, work);
    Val tv0{CPtr{tv.p, tv.s}, te[0], tc[0]};
    Val tv1{CPtr{tv.off(k.L).p, tv.s}, te[1], tc[1]};
    Val a0 = val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, idx);
    Val a1 = k.kind == DS_KIND_COMPLEX ? val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 1, k.L, idx) : a0;
    Out o0 = out_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, idx);
    Out o1 = out_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, k.ncomp - 1, k.L, idx);
    // add_rn reads a fully before writing (result goes to a's own slots):
    // stage a - t through scratch to avoid aliasing
    Ptr r0 = work.off(2 * (int64_t)k.L + 4);
    int32_t re0, re1;
    uint8_t rc0, rc1;
    ok &= add_rn(r0, &re0, &rc0, a0, tv0, true, k.L, k.p, work);
    if (k.kind == DS_KIND_COMPLEX) {
      Ptr r1 = r0.off(k.L);
      ok &= add_rn(r1, &re1, &rc1, a1, tv1, true, k.L, k.p, work);
      for (int l = 0; l < k.L; l++) o1.m[l] = r1[l];
      *o1.e = re1;
      *o1.c = rc1;
    }
    for (int l = 0; l < k.L; l++) o0.m[l] = r0[l];
    *o0.e = re0;
    *o0.c = rc0;
    if (!ok) atomicAdd(&k.status[2], 1);
  }
}

// signed minors for m = i+2 from local row (i+1): sig_k = RN(det * a_{i+1,k}),
// k < m-1, sig_{m-1} = det   (elim.py:56-61)
__global__ void k_emit_signed(KArgs k, int i) {
  if (k.status[0] >= 0) return;
  int m = i + 2;
  int64_t jl = (i + 1 - k.row_base) / k.world;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  Val d0 = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, 0, k.L, i);  // det_i (k_pivot / k_det_step)
  Val d1 = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, k.ncomp - 1, k.L, i);
  for (int64_t kk = tid; kk < m; kk += (int64_t)gridDim.x * blockDim.x) {
    int64_t oidx = mrow(k, jl) + kk;
    Out s0 = out_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, oidx);
    Out s1 = out_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, k.ncomp - 1, k.L, oidx);
    if (kk == m - 1) {
      set_val(s0, d0, k.L);
      if (k.kind == DS_KIND_COMPLEX) set_val(s1, d1, k.L);
      continue;
    }
    int64_t aidx = jl * k.n + kk;
    Val a0 = val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, aidx);
    Val a1 = k.kind == DS_KIND_COMPLEX ? val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 1, k.L, aidx) : a0;
    Ptr tmp = thread_scratch(k, tid);
    if (!g_mul(s0, s1, d0, d1, a0, a1, k.kind, k.L, k.p, tmp)) atomicAdd(&k.status[2], 1);
  }
}

// normalized = RN(sig_k / sig_0) unless sig_0 == 0 (elim.py:138-155)
__global__ void k_emit_norm(KArgs k, int i) {
  if (k.status[0] >= 0) return;
  int m = i + 2;
  int64_t jl = (i + 1 - k.row_base) / k.world;
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r0 = mrow(k, jl);
  Val l0 = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, r0);
  Val l1 = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, k.ncomp - 1, k.L, r0);
  bool lead_zero = is_zero_cls(l0.c) && (k.kind == DS_KIND_REAL || is_zero_cls(l1.c));
  if (tid == 0) k.row_flags[m - 1] = lead_zero ? 1 : 3;
  if (lead_zero) return;
  for (int64_t kk = tid; kk < m; kk += (int64_t)gridDim.x * blockDim.x) {
    int64_t idx = r0 + kk;
    Val s0 = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, idx);
    Val s1 = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, k.ncomp - 1, k.L, idx);
    Out o0 = out_at(k.nrm_limbs, k.nrm_exp, k.nrm_cls, k.m_count, 0, k.L, idx);
    Out o1 = out_at(k.nrm_limbs, k.nrm_exp, k.nrm_cls, k.m_count, k.ncomp - 1, k.L, idx);
    Ptr tmp = thread_scratch(k, tid);
    if (!g_div(o0, o1, s0, s1, l0, l1, k.kind, k.L, k.p, tmp, (unsigned int*)&k.status[3]))
      atomicAdd(&k.status[2], 1);
  }
}

// element-wise conformance op (ds_scalar_op)
__global__ void k_scalar_op(int op, int kind, int L, int p, int64_t count, const uint32_t* al, const int32_t* ae,
                            const uint8_t* ac, const uint32_t* bl, const int32_t* be, const uint8_t* bc,
                            uint32_t* ol, int32_t* oe, uint8_t* oc, uint32_t* scratch, int64_t sthreads,
                            int32_t* status) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int ncomp = kind == DS_KIND_COMPLEX ? 2 : 1;
  for (int64_t e = tid; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    Val a0 = val_at(al, ae, ac, count, 0, L, e), b0 = val_at(bl, be, bc, count, 0, L, e);
    Val a1 = kind ? val_at(al, ae, ac, count, 1, L, e) : a0;
    Val b1 = kind ? val_at(bl, be, bc, count, 1, L, e) : b0;
    Out o0 = out_at(ol, oe, oc, count, 0, L, e), o1 = out_at(ol, oe, oc, count, ncomp - 1, L, e);
    Ptr tmp{scratch + tid, sthreads};
    bool ok;
    switch (op) {
      case 0: ok = g_mul(o0, o1, a0, a1, b0, b1, kind, L, p, tmp); break;
      case 1: ok = g_sub(o0, o1, a0, a1, b0, b1, kind, L, p, tmp); break;
      case 2: ok = g_div(o0, o1, a0, a1, b0, b1, kind, L, p, tmp, (unsigned int*)&status[3]); break;
      default: ok = g_add(o0, o1, a0, a1, b0, b1, kind, L, p, tmp); break;
    }
    if (!ok) atomicAdd(&status[2], 1);
  }
}

// ---------------------------------------------------------------- warp division
// q = RN(a / b) for real scalars, one warp per quotient (ds_warpdiv.cuh).
// smem per warp: V (L) | U (nu + 32K) | Q (nu - L), nu = L + kq + 1.
__host__ __device__ static inline int wdiv_kq(int p) { return (p + 2 + 31) / 32; }
__host__ __device__ static inline int wdiv_words(int L, int p, int K) {
  int nu = L + wdiv_kq(p) + 1;
  return L + dsw::upad_words(nu + 32 * K) + (nu - L) + 4;
}

template <int K>
__device__ void wdiv_rn(Out o, const Val& a, const Val& b, int L, int p, uint32_t* sm, int32_t* status) {
  const int lane = threadIdx.x & 31;
  int neg = neg_of(a.c) ^ neg_of(b.c);
  if (is_zero_cls(a.c)) {
    for (int l = lane; l < L; l += 32) o.m[l] = 0u;
    if (lane == 0) {
      *o.e = 0;
      *o.c = zero_cls(neg);
    }
    return;
  }
  const int kq = wdiv_kq(p);
  const int nu = L + kq + 1;
  uint32_t* V = sm;
  uint32_t* U = V + L;
  uint32_t* Q = U + dsw::upad_words(nu + 32 * K);
  for (int l = lane; l < L; l += 32) V[l] = b.m[l];
  for (int k = lane; k < nu + 32 * K; k += 32) U[dsw::upad(k)] = (k >= kq && k < kq + L) ? a.m[k - kq] : 0u;
  uint32_t vb[K];
#pragma unroll
  for (int u = 0; u < K; u++) {
    int l = lane * K + u;
    vb[u] = l < L ? b.m[l] : 0u;
  }
  __syncwarp();
  bool rem = dsw::wdivrem<K>(Q, U, nu, V, vb, L);
  __syncwarp();
  int64_t e = dsw::wround(Q, nu - L, rem, a.e - b.e - 32 * (int64_t)kq, L, p, o.m.p, o.m.s);
  if (lane == 0) {
    *o.e = (int32_t)e;
    *o.c = nz_cls(neg);
    if (e < DS_EMIN || e > DS_EMAX) atomicAdd(&status[2], 1);
  }
}

// divisor_from_matrix (lookahead, world 1): the pivot a_ii is read from the
// matrix (row i is not staged yet); a zero pivot leaves everything untouched
// (the step's k_pivot_lite reports it)
template <int K>
__global__ void k_mult_w(KArgs k, int i, int jl0, int wwords, int divisor_from_matrix, const uint8_t* pscal) {
  extern __shared__ uint32_t wsm[];
  if (k.status[0] >= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (r >= k.nloc - jl0) return;
  PB pb = pb_view(k.pbuf, k.n, k.L, k.ncomp);
  Val b = pscal ? Val{CPtr{(const uint32_t*)pscal, 1}, *(const int32_t*)(pscal + 4 * k.L), pscal[4 * k.L + 4]}
          : divisor_from_matrix ? val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, (int64_t)i * k.n + i)
                                : val_at(pb.limbs, pb.exp, pb.cls, k.n, 0, k.L, i);
  if ((pscal || divisor_from_matrix) && is_zero_cls(b.c)) return;
  int64_t jl = jl0 + r;
  int64_t idx = jl * k.n + i;
  Val a = val_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, idx);
  Out z = out_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, 0, k.L, jl);
  wdiv_rn<K>(z, a, b, k.L, k.p, wsm + warp * wwords, k.status);
  __syncwarp();
  __threadfence_block();
  // a_ji <- -z_j (elim.py:53)
  Val zv = val_at(k.z_limbs, k.z_exp, k.z_cls, k.nloc, 0, k.L, jl);
  Out ao = out_at(k.a_limbs, k.a_exp, k.a_cls, k.a_count, 0, k.L, idx);
  for (int l = lane; l < k.L; l += 32) ao.m[l] = zv.m[l];
  if (lane == 0) {
    *ao.e = (int32_t)zv.e;
    uint8_t c = zv.c;
    *ao.c = (c == DS_CLS_POS) ? DS_CLS_NEG : (c == DS_CLS_NEG) ? DS_CLS_POS : (c == DS_CLS_PZERO) ? DS_CLS_NZERO : DS_CLS_PZERO;
  }
}

// multi-rank lookahead: the owner copies a_{i1,i1} (its local row jl) into the
// exchange buffer [L limbs | exp | cls] that is broadcast to every rank
__global__ void k_pscal_stage(KArgs k, int i1, int64_t jl, uint8_t* dst) {
  if (k.status[0] >= 0) return;
  const int64_t idx = jl * k.n + i1;
  for (int l = threadIdx.x; l < k.L; l += blockDim.x) ((uint32_t*)dst)[l] = k.a_limbs[(int64_t)l * k.a_count + idx];
  if (threadIdx.x == 0) {
    *(int32_t*)(dst + 4 * k.L) = k.a_exp[idx];
    dst[4 * k.L + 4] = k.a_cls[idx];
  }
}

template <int K>
__global__ void k_emit_norm_w(KArgs k, int i, int wwords) {
  extern __shared__ uint32_t wsm[];
  if (k.status[0] >= 0 && k.status[0] <= i) return;
  const int warp = threadIdx.x >> 5;
  int m = i + 2;
  int64_t jl = (i + 1 - k.row_base) / k.world;
  const int64_t kk = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t r0 = mrow(k, jl);
  Val l0 = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, r0);
  bool lead_zero = is_zero_cls(l0.c);
  if (blockIdx.x == 0 && threadIdx.x == 0) k.row_flags[m - 1] = lead_zero ? 1 : 3;
  if (lead_zero || kk >= m) return;
  int64_t idx = r0 + kk;
  Val s = val_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, 0, k.L, idx);
  Out o = out_at(k.nrm_limbs, k.nrm_exp, k.nrm_cls, k.m_count, 0, k.L, idx);
  wdiv_rn<K>(o, s, l0, k.L, k.p, wsm + warp * wwords, k.status);
}

// first step: det = piv (unrounded, elim.py:214); pivots[i] = piv; zero test
__global__ void k_pivot_lite(KArgs k, int i, int first) {
  if (k.status[0] >= 0) return;
  PB pb = pb_view(k.pbuf, k.n, k.L, k.ncomp);
  Val p0 = val_at(pb.limbs, pb.exp, pb.cls, k.n, 0, k.L, i);
  Val p1 = k.kind == DS_KIND_COMPLEX ? val_at(pb.limbs, pb.exp, pb.cls, k.n, 1, k.L, i) : p0;
  bool zero = is_zero_cls(p0.c) && (k.kind == DS_KIND_REAL || is_zero_cls(p1.c));
  __syncthreads();
  if (zero) {
    if (threadIdx.x == 0) k.status[0] = i;
    return;
  }
  for (int c = 0; c < k.ncomp; c++) {
    Val pv = val_at(pb.limbs, pb.exp, pb.cls, k.n, c, k.L, i);
    Out o = out_at(k.piv_limbs, k.piv_exp, k.piv_cls, k.n, c, k.L, i);
    Out d = out_at(k.det_limbs, k.det_exp, k.det_cls, k.n, c, k.L, i);
    for (int l = threadIdx.x; l < k.L; l += blockDim.x) {
      o.m[l] = pv.m[l];
      if (first) d.m[l] = pv.m[l];
    }
    if (threadIdx.x == 0) {
      *o.e = (int32_t)pv.e;
      *o.c = pv.c;
      if (first) {
        *d.e = (int32_t)pv.e;
        *d.c = pv.c;
      }
    }
  }
}

// sig_{m-1} = det_i (elim.py:60)
__global__ void k_emit_last(KArgs k, int i) {
  if (k.status[0] >= 0 && k.status[0] <= i) return;
  int64_t jl = (i + 1 - k.row_base) / k.world;
  int64_t idx = mrow(k, jl) + (i + 1);
  for (int c = 0; c < k.ncomp; c++) {
    Val d = val_at(k.det_limbs, k.det_exp, k.det_cls, k.n, c, k.L, i);
    Out o = out_at(k.sig_limbs, k.sig_exp, k.sig_cls, k.m_count, c, k.L, idx);
    for (int l = threadIdx.x; l < k.L; l += blockDim.x) o.m[l] = d.m[l];
    if (threadIdx.x == 0) {
      *o.e = (int32_t)d.e;
      *o.c = d.c;
    }
  }
}

// copy the seed det (ds_set_det) into det[i-1]'s role: det[i] = RN(seed * piv)
// is computed by mul_row_launch directly from `cur`.

// ---------------------------------------------------------------- host side
static int64_t general_scratch_words(int L, int kind) {
  int64_t w = 8 * (int64_t)L + 64;                        // real div / mul / add
  if (kind == DS_KIND_COMPLEX) w = cdiv_scratch_words(L, 32 * L) + 16;
  w += 6 * (int64_t)L + 16;                               // update: t (2L) + result (2L) + pad
  return w;
}

template <typename T>
static int dmalloc(ds_ctx* ctx, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    ctx->err = std::string("cudaMalloc failed: ") + cudaGetErrorString(e);
    g_last_error = ctx->err;
    return e == cudaErrorMemoryAllocation ? DS_OOM : DS_CUDA;
  }
  return DS_OK;
}

static int ensure_minors(ds_ctx* ctx) {
  if (ctx->sig_limbs) return DS_OK;
  const int64_t nc = ctx->ncomp, L = ctx->L, cnt = ctx->m_count;
  int rc;
  if ((rc = dmalloc(ctx, &ctx->sig_limbs, (size_t)(nc * L * cnt))) != DS_OK ||
      (rc = dmalloc(ctx, &ctx->sig_exp, (size_t)(nc * cnt))) != DS_OK ||
      (rc = dmalloc(ctx, &ctx->sig_cls, (size_t)(nc * cnt))) != DS_OK ||
      (rc = dmalloc(ctx, &ctx->nrm_limbs, (size_t)(nc * L * cnt))) != DS_OK ||
      (rc = dmalloc(ctx, &ctx->nrm_exp, (size_t)(nc * cnt))) != DS_OK ||
      (rc = dmalloc(ctx, &ctx->nrm_cls, (size_t)(nc * cnt))) != DS_OK)
    return rc;
  return DS_OK;
}

static void minors_free(ds_ctx* ctx) {
  void* ptrs[] = {ctx->sig_limbs, ctx->sig_exp, ctx->sig_cls, ctx->nrm_limbs, ctx->nrm_exp, ctx->nrm_cls};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  ctx->sig_limbs = ctx->nrm_limbs = nullptr;
  ctx->sig_exp = ctx->nrm_exp = nullptr;
  ctx->sig_cls = ctx->nrm_cls = nullptr;
}

static void stream_free(ds_ctx* ctx) {
  for (int st = 0; st < 2; st++) {
    for (int v = 0; v < 2; v++) {
      if (ctx->st_limbs[st][v]) cudaFreeHost(ctx->st_limbs[st][v]);
      if (ctx->st_exp[st][v]) cudaFreeHost(ctx->st_exp[st][v]);
      if (ctx->st_cls[st][v]) cudaFreeHost(ctx->st_cls[st][v]);
      ctx->st_limbs[st][v] = nullptr;
      ctx->st_exp[st][v] = nullptr;
      ctx->st_cls[st][v] = nullptr;
    }
    if (ctx->st_flags[st]) cudaFreeHost(ctx->st_flags[st]);
    ctx->st_flags[st] = nullptr;
    if (ctx->st_ev[st]) cudaEventDestroy(ctx->st_ev[st]);
    ctx->st_ev[st] = nullptr;
  }
  ctx->st_batch = 0;
}

extern "C" {

const char* ds_version(void) { return DS_VERSION; }

const char* ds_last_error(ds_ctx* ctx) { return ctx ? ctx->err.c_str() : g_last_error.c_str(); }

void* ds_stream(ds_ctx* ctx) { return (void*)ctx->stream; }

int ds_set_stream(ds_ctx* ctx, void* stream) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  return DS_OK;
}

int ds_use_pivot_buffer(ds_ctx* ctx, void* dptr, size_t bytes) {
  if (dptr && bytes < ctx->pbuf_bytes) return DS_INVALID;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->pbuf = dptr ? (uint8_t*)dptr : ctx->own_pbuf;
  return DS_OK;
}

int ds_pivot_copy(ds_ctx* dst, ds_ctx* src) {
  ds_ctx* ctx = dst;
  if (dst->pbuf_bytes != src->pbuf_bytes) return DS_INVALID;
  CK(cudaSetDevice(src->device));
  CK(cudaEventRecord(src->ev, src->stream));
  CK(cudaSetDevice(dst->device));
  CK(cudaStreamWaitEvent(dst->stream, src->ev, 0));
  if (dst->device == src->device) {
    CK(cudaMemcpyAsync(dst->pbuf, src->pbuf, dst->pbuf_bytes, cudaMemcpyDeviceToDevice, dst->stream));
  } else {
    CK(cudaMemcpyPeerAsync(dst->pbuf, dst->device, src->pbuf, src->device, dst->pbuf_bytes, dst->stream));
  }
  // src must not overwrite its buffer before the copy has read it
  CK(cudaEventRecord(dst->ev, dst->stream));
  CK(cudaSetDevice(src->device));
  CK(cudaStreamWaitEvent(src->stream, dst->ev, 0));
  return DS_OK;
}

int64_t ds_launch_count(ds_ctx* ctx) { return ctx->launches; }

static int ds_create_sized(ds_ctx** out, int n, long prec_bits, int kind, int device, int rank, int world,
                           int nloc_override);

int ds_create_block(ds_ctx** out, int n, long prec_bits, int kind, int device, int row0, int nrows) {
  *out = nullptr;
  if (row0 < 0 || nrows < 1 || row0 + nrows > n) return DS_INVALID;
  // a one-rank context sized for the block, then re-based onto rows [row0, row0 + nrows)
  int rc = ds_create_sized(out, n, prec_bits, kind, device, 0, 1, nrows);
  if (rc != DS_OK) return rc;
  (*out)->row_base = row0;
  return DS_OK;
}

int ds_pivot_load(ds_ctx* ctx, int step, const ds_soa* row) {
  if (step < 0 || step >= ctx->n || row->count != ctx->n) return DS_INVALID;
  CK(cudaSetDevice(ctx->device));
  const int n = ctx->n, L = ctx->L, nc = ctx->ncomp;
  PB pb = pb_view(ctx->pbuf, n, L, nc);
  // the host row is a count-n SoA: exactly the pivot buffer's planes
  CK(cudaMemcpyAsync(pb.limbs, row->limbs, sizeof(uint32_t) * nc * L * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(pb.exp, row->exp, sizeof(int32_t) * nc * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(pb.cls, row->cls, (size_t)nc * n, cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += (int64_t)nc * (4 * L + 5) * n;
  (void)step;
  return DS_OK;
}

void ds_destroy(ds_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  // ctx->z_* alias one of the two multiplier buffers: free those by their own pointers
  void* ptrs[] = {ctx->a_limbs, ctx->a_exp, ctx->a_cls, ctx->own_pbuf, ctx->zb_limbs[0], ctx->zb_exp[0], ctx->zb_cls[0],
                  ctx->piv_limbs, ctx->det_limbs, ctx->cur_limbs, ctx->piv_exp, ctx->det_exp, ctx->cur_exp,
                  ctx->piv_cls, ctx->det_cls, ctx->cur_cls, ctx->sig_limbs, ctx->nrm_limbs, ctx->sig_exp,
                  ctx->nrm_exp, ctx->sig_cls, ctx->nrm_cls, ctx->row_flags, ctx->status, ctx->scratch, ctx->swaps, ctx->pbest};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  void* zb1[] = {ctx->zb_limbs[1], ctx->zb_exp[1], ctx->zb_cls[1]};
  for (void* p : zb1)
    if (p) cudaFree(p);
  if (ctx->la) {
    cudaStreamSynchronize(ctx->la);
    cudaStreamDestroy(ctx->la);
  }
  update_plan_free(&ctx->plan);
  tc_plan_free(&ctx->tc);
  if (ctx->side) cudaStreamSynchronize(ctx->side);
  if (ctx->scratch_side) cudaFree(ctx->scratch_side);
  if (ctx->ws_dx) cudaFree(ctx->ws_dx);
  if (ctx->ws_dy) cudaFree(ctx->ws_dy);
  if (ctx->ws_ex) cudaFree(ctx->ws_ex);
  if (ctx->ws_ey) cudaFree(ctx->ws_ey);
  if (ctx->ev_piv) cudaEventDestroy(ctx->ev_piv);
  if (ctx->ev_upd) cudaEventDestroy(ctx->ev_upd);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->snap_limbs) cudaFree(ctx->snap_limbs);
  if (ctx->snap_exp) cudaFree(ctx->snap_exp);
  if (ctx->snap_cls) cudaFree(ctx->snap_cls);
  for (cudaEvent_t ev : ctx->prof_ev) cudaEventDestroy(ev);
  stream_free(ctx);
  if (ctx->ev) cudaEventDestroy(ctx->ev);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int ds_create(ds_ctx** out, int n, long prec_bits, int kind, int device, int rank, int world) {
  return ds_create_sized(out, n, prec_bits, kind, device, rank, world, -1);
}

static int ds_create_sized(ds_ctx** out, int n, long prec_bits, int kind, int device, int rank, int world,
                           int nloc_override) {
  *out = nullptr;
  if (n < 1 || prec_bits < 64 || prec_bits > (1L << 24) || (kind != DS_KIND_REAL && kind != DS_KIND_COMPLEX) ||
      world < 1 || rank < 0 || rank >= world) {
    g_last_error = "ds_create: invalid arguments";
    return DS_INVALID;
  }
  ds_ctx* ctx = new ds_ctx();
  ctx->n = n; ctx->p = (int)prec_bits; ctx->L = nlimbs(prec_bits); ctx->kind = kind;
  ctx->ncomp = kind == DS_KIND_COMPLEX ? 2 : 1; ctx->device = device; ctx->rank = rank; ctx->world = world;
  ctx->nloc = nloc_override >= 0 ? nloc_override : (n - rank + world - 1) / world;
  ctx->row_base = 0;
  ctx->launches = 0;
  memset(&ctx->plan, 0, sizeof(ctx->plan));
  CK(cudaSetDevice(device));
  // the elimination's critical path (pivot -> multipliers -> update) runs at the
  // highest stream priority, the outputs-only side stream (det chain, minors
  // emission) at the lowest: pending update CTAs get SMs before emission blocks
  // (numerically lower = higher priority): lookahead > main > side
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  const int prio_main = prio_hi < prio_lo ? prio_hi + 1 : prio_hi;
  CK(cudaStreamCreateWithPriority(&ctx->own_stream, cudaStreamNonBlocking, prio_main));
  ctx->stream = ctx->own_stream;
  CK(cudaEventCreateWithFlags(&ctx->ev, cudaEventDisableTiming));
  CK(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, prio_lo));
  CK(cudaStreamCreateWithPriority(&ctx->la, cudaStreamNonBlocking, prio_hi));
  CK(cudaEventCreateWithFlags(&ctx->ev_prep, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_a, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_mult, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_la_done, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_piv, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_upd, cudaEventDisableTiming));
  int L = ctx->L, nc = ctx->ncomp;
  // plane stride padded to 32 elements (128 B): keeps every limb plane 16-byte aligned for the tile tensor map
  ctx->a_count = (((int64_t)ctx->nloc * n) + 31) & ~(int64_t)31;
  int rc;
#define AL(ptr, cnt) if ((rc = dmalloc(ctx, &ptr, (size_t)(cnt))) != DS_OK) { ds_destroy(ctx); return rc; }
  AL(ctx->a_limbs, (int64_t)nc * L * ctx->a_count);
  AL(ctx->a_exp, (int64_t)nc * ctx->a_count);
  AL(ctx->a_cls, (int64_t)nc * ctx->a_count);
  ctx->pbuf_bytes = pbuf_size(n, L, nc);
  AL(ctx->own_pbuf, ctx->pbuf_bytes);
  ctx->pbuf = ctx->own_pbuf;
  AL(ctx->zb_limbs[0], (int64_t)nc * L * ctx->nloc);
  AL(ctx->zb_exp[0], (int64_t)nc * ctx->nloc);
  AL(ctx->zb_cls[0], (int64_t)nc * ctx->nloc);
  AL(ctx->zb_limbs[1], (int64_t)nc * L * ctx->nloc);
  AL(ctx->zb_exp[1], (int64_t)nc * ctx->nloc);
  AL(ctx->zb_cls[1], (int64_t)nc * ctx->nloc);
  ctx->z_limbs = ctx->zb_limbs[0];
  ctx->z_exp = ctx->zb_exp[0];
  ctx->z_cls = ctx->zb_cls[0];
  ctx->la_step = -1;
  ctx->la_limit = -1;
  AL(ctx->piv_limbs, (int64_t)nc * L * n); AL(ctx->piv_exp, (int64_t)nc * n); AL(ctx->piv_cls, (int64_t)nc * n);
  AL(ctx->det_limbs, (int64_t)nc * L * n); AL(ctx->det_exp, (int64_t)nc * n); AL(ctx->det_cls, (int64_t)nc * n);
  AL(ctx->cur_limbs, (int64_t)nc * L); AL(ctx->cur_exp, nc); AL(ctx->cur_cls, nc);
  // minors storage is allocated on first use (ensure_minors): all owned rows, or
  // the ring set up by ds_stream_minors
  ctx->m_rows = ctx->nloc > 0 ? ctx->nloc : 1;
  ctx->m_count = ctx->a_count > 0 ? ctx->a_count : 32;
  AL(ctx->row_flags, n);
  AL(ctx->status, 8);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  ctx->scratch_threads = (int64_t)sms * 4 * 128;
  ctx->scratch_words = general_scratch_words(L, kind);
  AL(ctx->scratch, ctx->scratch_threads * ctx->scratch_words);
#undef AL
  CK(cudaMemsetAsync(ctx->row_flags, 0, n, ctx->stream));
  int32_t st[8] = {-1, 0, 0, 0, 0, 0, 0, 0};
  CK(cudaMemcpyAsync(ctx->status, st, sizeof(st), cudaMemcpyHostToDevice, ctx->stream));
  if (kind == DS_KIND_REAL) {
    rc = update_plan_init(&ctx->plan, n, ctx->p, device);
    if (rc != DS_OK) {
      ctx->err = g_last_error;
      ds_destroy(ctx);
      return rc;
    }
    if (ctx->plan.enabled) {
      rc = tc_plan_init(&ctx->tc, n, ctx->nloc, ctx->p, device);
      if (rc != DS_OK) {
        ctx->err = "tensor-core update plan: device allocation or attribute failed";
        ds_destroy(ctx);
        return rc;
      }
      size_t a1 = mul_ws_doubles(&ctx->plan, 1), an = mul_ws_doubles(&ctx->plan, n);
      if ((rc = dmalloc(ctx, &ctx->ws_dx, a1)) != DS_OK || (rc = dmalloc(ctx, &ctx->ws_dy, a1)) != DS_OK ||
          (rc = dmalloc(ctx, &ctx->ws_ex, a1)) != DS_OK || (rc = dmalloc(ctx, &ctx->ws_ey, an)) != DS_OK) {
        ds_destroy(ctx);
        return rc;
      }
    }
  }
  if (kind == DS_KIND_COMPLEX) {
    rc = tc_plan_init_c(&ctx->tc, n, ctx->nloc, ctx->p, device);
    if (rc != DS_OK) {
      ctx->err = "complex tensor-core update plan: device allocation or attribute failed";
      ds_destroy(ctx);
      return rc;
    }
    if (ctx->tc.enabled &&
        cudaMalloc(&ctx->scratch_side, sizeof(uint32_t) * ctx->scratch_threads * ctx->scratch_words) != cudaSuccess) {
      ctx->scratch_side = nullptr;
      ds_destroy(ctx);
      return DS_OOM;
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  *out = ctx;
  return DS_OK;
}

// host matrix layouts accepted by ds_load / ds_fetch / ds_results_fetch: the
// full n x n matrix (count n*n; this rank's row jl is global row rank +
// jl*world) or only the rows this rank owns (count nloc*n, row jl at jl*n).
// Returns the first host row and the host row stride of local row 0, 1, ...
static bool host_rows(const ds_ctx* ctx, int64_t count, int64_t* r0, int64_t* rs) {
  const int64_t n = ctx->n;
  if (count == n * n) {
    *r0 = ctx->row_base + ctx->rank;
    *rs = ctx->world;
    return true;
  }
  if (count == (int64_t)ctx->nloc * n) {
    *r0 = 0;
    *rs = 1;
    return true;
  }
  return false;
}

// fresh run state after new matrix contents (ds_load, ds_generate)
static int reset_run_state(ds_ctx* ctx) {
  const int n = ctx->n;
  ctx->host_have_det = 0;
  ctx->la_step = -1;
  ctx->det_from_cur = 0;
  CK(cudaMemsetAsync(ctx->row_flags, 0, n, ctx->stream));
  if (ctx->swaps) CK(cudaMemsetAsync(ctx->swaps, 0, n, ctx->stream));
  int32_t st[8] = {-1, 0, 0, 0, 0, 0, 0, 0};
  CK(cudaMemcpyAsync(ctx->status, st, sizeof(st), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->st_next = 1;
  ctx->st_pending = 0;
  return DS_OK;
}

static int copy_row_range_to(ds_ctx* ctx, ds_soa* dst, const uint32_t* limbs, const int32_t* ex, const uint8_t* cl,
                             int r0, int r1, int width, cudaStream_t s, int hrow0);

// ---- streaming of minors rows (ds_stream_minors / ds_stream_flush)
int ds_stream_minors(ds_ctx* ctx, int batch_steps, ds_rows_cb cb, void* user) {
  if (ctx->row_base != 0 && batch_steps > 0) {
    ctx->err = "minors streaming is not available on a row-block (paged) context";
    return DS_INVALID;
  }
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaStreamSynchronize(ctx->side));
  stream_free(ctx);
  int ring = ctx->nloc > 0 ? ctx->nloc : 1;
  const int per = batch_steps > 0 ? batch_steps / ctx->world + 2 : 0;
  if (batch_steps > 0 && cb) ring = std::min(ring, 3 * per);
  if (ring != ctx->m_rows) {
    minors_free(ctx);
    ctx->m_rows = ring;
    ctx->m_count = (((int64_t)ring * ctx->n) + 31) & ~(int64_t)31;
  }
  if (batch_steps <= 0 || !cb) return DS_OK;
  const size_t cnt = (size_t)per * ctx->n, nc = ctx->ncomp, L = ctx->L;
  for (int st = 0; st < 2; st++) {
    for (int v = 0; v < 2; v++) {
      if (cudaMallocHost((void**)&ctx->st_limbs[st][v], sizeof(uint32_t) * nc * L * cnt) != cudaSuccess ||
          cudaMallocHost((void**)&ctx->st_exp[st][v], sizeof(int32_t) * nc * cnt) != cudaSuccess ||
          cudaMallocHost((void**)&ctx->st_cls[st][v], nc * cnt) != cudaSuccess) {
        cudaGetLastError();
        stream_free(ctx);
        ctx->err = "pinned staging for the minors stream could not be allocated";
        return DS_OOM;
      }
    }
    CK(cudaMallocHost((void**)&ctx->st_flags[st], (size_t)per));
    CK(cudaEventCreateWithFlags(&ctx->st_ev[st], cudaEventDisableTiming));
  }
  ctx->st_rows_cap = per;
  ctx->st_batch = batch_steps;
  ctx->st_cb = cb;
  ctx->st_user = user;
  ctx->st_next = 1;
  ctx->st_pending = 0;
  return DS_OK;
}

static void st_deliver(ds_ctx* ctx, int set, int g0, int nrows) {
  const int64_t cnt = (int64_t)ctx->st_rows_cap * ctx->n;
  ds_soa sg{ctx->st_limbs[set][0], ctx->st_exp[set][0], ctx->st_cls[set][0], cnt};
  ds_soa nm{ctx->st_limbs[set][1], ctx->st_exp[set][1], ctx->st_cls[set][1], cnt};
  ctx->st_cb(g0, ctx->world, nrows, &sg, &nm, ctx->st_flags[set], ctx->st_user);
}

int ds_stream_flush(ds_ctx* ctx, int upto_step, int final) {
  if (!ctx->st_batch) return DS_OK;
  CK(cudaSetDevice(ctx->device));
  const int n = ctx->n, world = ctx->world, rank = ctx->rank;
  // global rows g in [st_next, hi] are final after steps [0, upto_step)
  const int hi = std::min(upto_step, n - 1);
  int jl_a = ctx->st_next <= rank ? 0 : (ctx->st_next - rank + world - 1) / world;
  int jl_b = hi < rank ? 0 : (hi - rank) / world + 1;
  if (jl_b < jl_a) jl_b = jl_a;
  const int nrows = jl_b - jl_a;
  if (nrows > ctx->st_rows_cap) {
    ctx->err = "ds_stream_flush: more rows finalised since the last flush than the stream batch allows";
    return DS_INVALID;
  }
  int set = ctx->st_pending ? ctx->st_set ^ 1 : ctx->st_set;
  const int g0 = rank + jl_a * world;
  if (nrows > 0 && ctx->sig_limbs) {
    // emission may have run on either stream: the copies (side stream) follow both
    CK(cudaEventRecord(ctx->ev, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev, 0));
    const int width = rank + (jl_b - 1) * world + 1;
    const int64_t cnt = (int64_t)ctx->st_rows_cap * n;
    ds_soa sg{ctx->st_limbs[set][0], ctx->st_exp[set][0], ctx->st_cls[set][0], cnt};
    ds_soa nm{ctx->st_limbs[set][1], ctx->st_exp[set][1], ctx->st_cls[set][1], cnt};
    int rc;
    if ((rc = copy_row_range_to(ctx, &sg, ctx->sig_limbs, ctx->sig_exp, ctx->sig_cls, jl_a, jl_b, width, ctx->side,
                                0)) != DS_OK ||
        (rc = copy_row_range_to(ctx, &nm, ctx->nrm_limbs, ctx->nrm_exp, ctx->nrm_cls, jl_a, jl_b, width, ctx->side,
                                0)) != DS_OK)
      return rc;
    CK(cudaMemcpy2DAsync(ctx->st_flags[set], 1, ctx->row_flags + g0, world, 1, nrows, cudaMemcpyDeviceToHost,
                         ctx->side));
    ctx->d2h_bytes += nrows;
    CK(cudaEventRecord(ctx->st_ev[set], ctx->side));
  }
  // hand the previous batch to the caller while this one copies
  if (ctx->st_pending) {
    const int old = ctx->st_set;
    CK(cudaEventSynchronize(ctx->st_ev[old]));
    st_deliver(ctx, old, ctx->st_pend_g0, ctx->st_pend_rows);
    ctx->st_pending = 0;
  }
  if (nrows > 0 && ctx->sig_limbs) {
    ctx->st_set = set;
    ctx->st_pending = 1;
    ctx->st_pend_g0 = g0;
    ctx->st_pend_rows = nrows;
  }
  if (hi + 1 > ctx->st_next) ctx->st_next = hi + 1;
  if (final && ctx->st_pending) {
    CK(cudaEventSynchronize(ctx->st_ev[ctx->st_set]));
    st_deliver(ctx, ctx->st_set, ctx->st_pend_g0, ctx->st_pend_rows);
    ctx->st_pending = 0;
  }
  return DS_OK;
}

int ds_load(ds_ctx* ctx, const ds_soa* h) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->side));
  int n = ctx->n, L = ctx->L;
  int64_t r0, rs;
  if (!host_rows(ctx, h->count, &r0, &rs)) return DS_INVALID;
  // gather owned rows (row-cyclic) plane by plane; contiguous when world == 1
  // or when the caller passes only its owned rows
  for (int c = 0; c < ctx->ncomp; c++) {
    for (int l = 0; l < L; l++) {
      const uint32_t* src = h->limbs + ((int64_t)c * L + l) * h->count;
      uint32_t* dst = ctx->a_limbs + ((int64_t)c * L + l) * ctx->a_count;
      if (rs == 1) {
        CK(cudaMemcpyAsync(dst, src, sizeof(uint32_t) * ctx->nloc * n, cudaMemcpyHostToDevice, ctx->stream));
      } else {
        CK(cudaMemcpy2DAsync(dst, sizeof(uint32_t) * n, src + r0 * n, sizeof(uint32_t) * n * rs,
                             sizeof(uint32_t) * n, ctx->nloc, cudaMemcpyHostToDevice, ctx->stream));
      }
    }
    const int32_t* se = h->exp + (int64_t)c * h->count;
    const uint8_t* sc = h->cls + (int64_t)c * h->count;
    CK(cudaMemcpy2DAsync(ctx->a_exp + (int64_t)c * ctx->a_count, sizeof(int32_t) * n, se + r0 * n,
                         sizeof(int32_t) * n * rs, sizeof(int32_t) * n, ctx->nloc, cudaMemcpyHostToDevice,
                         ctx->stream));
    CK(cudaMemcpy2DAsync(ctx->a_cls + (int64_t)c * ctx->a_count, n, sc + r0 * n, (size_t)n * rs,
                         n, ctx->nloc, cudaMemcpyHostToDevice, ctx->stream));
  }
  ctx->h2d_bytes += (int64_t)ctx->ncomp * (4 * L + 5) * ctx->nloc * n;
  return reset_run_state(ctx);
}

// ds_load without the run-state reset: the rows a step hook edited go back to
// the device mid-run (elim.eliminate with step_hook)
int ds_update_rows(ds_ctx* ctx, const ds_soa* h) {
  const int have = ctx->host_have_det, dfc = ctx->det_from_cur;
  const int nxt = ctx->st_next, pend = ctx->st_pending;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->side));
  int n = ctx->n, L = ctx->L;
  int64_t r0, rs;
  if (!host_rows(ctx, h->count, &r0, &rs)) return DS_INVALID;
  for (int c = 0; c < ctx->ncomp; c++) {
    for (int l = 0; l < L; l++)
      CK(cudaMemcpy2DAsync(ctx->a_limbs + ((int64_t)c * L + l) * ctx->a_count, sizeof(uint32_t) * n,
                           h->limbs + ((int64_t)c * L + l) * h->count + r0 * n, sizeof(uint32_t) * n * rs,
                           sizeof(uint32_t) * n, ctx->nloc, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpy2DAsync(ctx->a_exp + (int64_t)c * ctx->a_count, sizeof(int32_t) * n, h->exp + (int64_t)c * h->count + r0 * n,
                         sizeof(int32_t) * n * rs, sizeof(int32_t) * n, ctx->nloc, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpy2DAsync(ctx->a_cls + (int64_t)c * ctx->a_count, n, h->cls + (int64_t)c * h->count + r0 * n, (size_t)n * rs,
                         n, ctx->nloc, cudaMemcpyHostToDevice, ctx->stream));
  }
  ctx->h2d_bytes += (int64_t)ctx->ncomp * (4 * L + 5) * ctx->nloc * n;
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->host_have_det = have;
  ctx->det_from_cur = dfc;
  ctx->st_next = nxt;
  ctx->st_pending = pend;
  ctx->la_step = -1;  // multipliers computed ahead from the old rows are stale
  return DS_OK;
}

int gen_uniform_launch(cudaStream_t s, uint32_t* limbs, int32_t* ex, uint8_t* cl, int64_t count, int n, int L, int p,
                       int rank, int world, int nloc, uint64_t seed);

int ds_generate(ds_ctx* ctx, int family, uint64_t seed) {
  if (family != DS_FAMILY_RANDOM_UNIFORM || ctx->kind != DS_KIND_REAL) {
    ctx->err = "ds_generate: only the real random_uniform family is generated on the device";
    return DS_INVALID;
  }
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->side));
  if (gen_uniform_launch(ctx->stream, ctx->a_limbs, ctx->a_exp, ctx->a_cls, ctx->a_count, ctx->n, ctx->L, ctx->p,
                         ctx->row_base + ctx->rank, ctx->world, ctx->nloc, seed) != 0) {
    ctx->err = "k_gen_uniform launch failed";
    return DS_CUDA;
  }
  ctx->launches++;
  return reset_run_state(ctx);
}

int ds_fetch(ds_ctx* ctx, ds_soa* h) {
  CK(cudaSetDevice(ctx->device));
  int n = ctx->n, L = ctx->L;
  int64_t r0, rs;
  if (!host_rows(ctx, h->count, &r0, &rs)) return DS_INVALID;
  for (int c = 0; c < ctx->ncomp; c++) {
    for (int l = 0; l < L; l++) {
      uint32_t* dst = h->limbs + ((int64_t)c * L + l) * h->count;
      const uint32_t* src = ctx->a_limbs + ((int64_t)c * L + l) * ctx->a_count;
      CK(cudaMemcpy2DAsync(dst + r0 * n, sizeof(uint32_t) * n * rs, src, sizeof(uint32_t) * n,
                           sizeof(uint32_t) * n, ctx->nloc, cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaMemcpy2DAsync(h->exp + (int64_t)c * h->count + r0 * n, sizeof(int32_t) * n * rs,
                         ctx->a_exp + (int64_t)c * ctx->a_count, sizeof(int32_t) * n, sizeof(int32_t) * n, ctx->nloc,
                         cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpy2DAsync(h->cls + (int64_t)c * h->count + r0 * n, (size_t)n * rs,
                         ctx->a_cls + (int64_t)c * ctx->a_count, n, n, ctx->nloc, cudaMemcpyDeviceToHost, ctx->stream));
  }
  ctx->d2h_bytes += (int64_t)ctx->ncomp * (4 * L + 5) * ctx->nloc * n;
  CK(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_pivot_buffer(ds_ctx* ctx, void** dptr, size_t* bytes) {
  *dptr = ctx->pbuf;
  *bytes = ctx->pbuf_bytes;
  return DS_OK;
}

static int grid_for(ds_ctx* ctx, int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  int64_t gmax = ctx->scratch_threads / block;
  if (g > gmax) g = gmax;
  if (g < 1) g = 1;
  return (int)g;
}

int ds_pivot_stage(ds_ctx* ctx, int i) {
  if (i < 0 || i >= ctx->n || !owns_row(ctx, i)) return DS_INVALID;
  CK(cudaSetDevice(ctx->device));
  KArgs k = kargs(ctx);
  int64_t tot = (int64_t)ctx->ncomp * (ctx->L + 2) * ctx->n;
  int g = (int)((tot + 255) / 256);
  if (g > 148 * 16) g = 148 * 16;
  k_stage<<<g, 256, 0, ctx->stream>>>(k, i);
  ctx->launches++;
  CK(cudaGetLastError());
  return DS_OK;
}

// use the general engine for the real update too (testing / A-B checks)
static int g_force_general = -1;
static bool force_general() {
  if (g_force_general < 0) {
    const char* s = getenv("DS_FORCE_GENERAL_UPDATE");
    g_force_general = (s && s[0] == '1') ? 1 : 0;
  }
  return g_force_general == 1;
}

// limbs per lane of the warp division: the smallest instantiated K with 32 K >= L
// (33,220 bits = 1039 limbs takes K = 36, not 64: half the lane work, no spills)
static int warp_k(int L) {
  static const int ks[] = {1, 2, 4, 8, 16, 24, 32, 36, 48, 64};
  for (int K : ks)
    if (32 * K >= L) return K;
  return 64;
}

#define WDIV_DISPATCH(K_, KERNEL, grid, block, smem, s, ...)                 \
  switch (K_) {                                                              \
    case 1: KERNEL<1><<<grid, block, smem, s>>>(__VA_ARGS__); break;         \
    case 2: KERNEL<2><<<grid, block, smem, s>>>(__VA_ARGS__); break;         \
    case 4: KERNEL<4><<<grid, block, smem, s>>>(__VA_ARGS__); break;         \
    case 8: KERNEL<8><<<grid, block, smem, s>>>(__VA_ARGS__); break;         \
    case 16: KERNEL<16><<<grid, block, smem, s>>>(__VA_ARGS__); break;       \
    case 24: KERNEL<24><<<grid, block, smem, s>>>(__VA_ARGS__); break;       \
    case 32: KERNEL<32><<<grid, block, smem, s>>>(__VA_ARGS__); break;       \
    case 36: KERNEL<36><<<grid, block, smem, s>>>(__VA_ARGS__); break;       \
    case 48: KERNEL<48><<<grid, block, smem, s>>>(__VA_ARGS__); break;       \
    default: KERNEL<64><<<grid, block, smem, s>>>(__VA_ARGS__); break;       \
  }

static bool fast_real(ds_ctx* ctx) {
  // the fused update or a tensor-core update, plus the DFMA row products
  return ctx->kind == DS_KIND_REAL && ctx->plan.enabled && (ctx->plan.fused || ctx->tc.enabled) &&
         !force_general();
}

// the warp division holds K = L/32 <= 64 limbs per lane in registers (K = 64:
// 33220 bits, L = 1039); wider precisions divide with the thread-level engine
static bool wdiv_ok(const ds_ctx* ctx) { return ctx->L <= 2048; }

static void set_wdiv_attrs(int maxsm) {
  static bool done = false;
  if (done) return;
  done = true;
#define SA(KERNEL) \
  cudaFuncSetAttribute(KERNEL<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<36>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<48>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm); \
  cudaFuncSetAttribute(KERNEL<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  SA(k_mult_w)
  SA(k_emit_norm_w)
#undef SA
}

// shared-memory scratch for the thread-level complex kernels: threads per block
// = how many per-thread scratch areas fit (<= 8, and no more than the work
// items); 0 when one does not fit (very wide precisions: global scratch)
static size_t cx_smem_launch(ds_ctx* ctx, KArgs* k, int64_t work) {
  static int maxsm = 0;
  static bool attrs = false;
  if (!maxsm) cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  const size_t per = sizeof(uint32_t) * ((size_t)ctx->scratch_words + 4 * (size_t)ctx->L);  // scratch + 4 operands
  int t = per ? (int)((size_t)maxsm / per) : 0;
  if (t > 8) t = 8;
  if (work < t) t = (int)(work > 0 ? work : 1);
  if (t < 1 || getenv("DS_CX_GLOBAL_SCRATCH")) {
    k->sm_threads = 0;
    return 0;
  }
  if (!attrs) {
    cudaFuncSetAttribute(k_det_step, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
    cudaFuncSetAttribute(k_mult_c2, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
    cudaFuncSetAttribute(k_emit_signed_c2, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
    cudaFuncSetAttribute(k_emit_norm_c2, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
    attrs = true;
  }
  k->sm_threads = t;
  return per * (size_t)t;
}

// warps per block of the warp-level complex kernels (0: their region does not fit
// in shared memory -- wide precisions keep the thread-level kernels)
static int cw_plan(ds_ctx* ctx, int* words) {
  static int maxsm = 0;
  static bool attrs = false;
  static int dyn_max = 0;  // opt-in maximum minus the kernels' static shared memory
  if (!maxsm) {
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
    dyn_max = maxsm - 4096;
  }
  const int64_t w = dscw::warp_words(ctx->L, ctx->p);
  *words = (int)w;
  if (getenv("DS_CX_THREAD")) return 0;
  int64_t wpb = (int64_t)dyn_max / (4 * w);
  if (wpb > 8) wpb = 8;
  if (wpb < 1 || ctx->L > 512) return 0;
  if (!attrs) {
    bool ok = cudaFuncSetAttribute(k_cw_det, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) == cudaSuccess &&
              cudaFuncSetAttribute(k_cw_mult, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) == cudaSuccess &&
              cudaFuncSetAttribute(k_cw_emit_signed, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) ==
                  cudaSuccess &&
              cudaFuncSetAttribute(k_cw_emit_norm, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max) ==
                  cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      dyn_max = 48 * 1024;  // the default limit: fewer warps per block
      wpb = (int64_t)dyn_max / (4 * w);
      if (wpb < 1) return 0;
    }
    attrs = true;
  }
  return (int)wpb;
}

int ds_step(ds_ctx* ctx, int i, int collect_minors, int series) {
  if (i < 0 || i >= ctx->n) return DS_INVALID;
  CK(cudaSetDevice(ctx->device));
  // multipliers of step i live in z buffer i & 1 (the lookahead fills the other)
  ctx->z_limbs = ctx->zb_limbs[i & 1];
  ctx->z_exp = ctx->zb_exp[i & 1];
  ctx->z_cls = ctx->zb_cls[i & 1];
  const bool la_have = ctx->la_step == i;
  ctx->la_step = -1;
  KArgs k = kargs(ctx);
  cudaStream_t s = ctx->stream;
  const bool fast = fast_real(ctx);
  const int L = ctx->L, n = ctx->n;
  const int K = warp_k(L);
  const int wwords = wdiv_words(L, ctx->p, K);
  const int wpb = 4;  // warps per block for the division kernels
  if (fast) {
    int maxsm = 0;
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
    set_wdiv_attrs(maxsm);
  }
  PB pb = pb_view(ctx->pbuf, n, L, ctx->ncomp);
  // complex on the tensor cores: det chain and minors (general kernels) on the side
  // stream with their own scratch, off the update's critical path
  const bool cxf = ctx->kind == DS_KIND_COMPLEX && ctx->tc.enabled && ctx->scratch_side && !force_general();
  KArgs ks = k;
  ks.scratch = ctx->scratch_side;
  // ---- pivot: zero test, pivots[i], det chain (elim.py:209-215)
  if (cxf) {
    int first = ctx->host_have_det ? 0 : 1;
    k_pivot_lite<<<1, 128, 0, s>>>(k, i, first);
    ctx->launches++;
    if (!first) {
      CK(cudaEventRecord(ctx->ev_piv, s));
      CK(cudaStreamWaitEvent(ctx->side, ctx->ev_piv, 0));
      int cw_words = 0;
      const int cw_wpb = cw_plan(ctx, &cw_words);
      if (cw_wpb >= 2) {  // one warp per component
        k_cw_det<<<1, 64, (size_t)2 * cw_words * 4, ctx->side>>>(ks, i, ctx->det_from_cur, cw_words);
      } else {
        KArgs kd = ks;
        const size_t sm = cx_smem_launch(ctx, &kd, 1);
        k_det_step<<<1, kd.sm_threads ? 1 : 32, sm, ctx->side>>>(kd, i, ctx->det_from_cur);
      }
      ctx->launches++;
    }
  } else if (fast) {
    int first = ctx->host_have_det ? 0 : 1;
    k_pivot_lite<<<1, 128, 0, s>>>(k, i, first);
    ctx->launches++;
    if (!first) {
      // det_i = RN(det_{i-1} * piv_i) on the side stream, from pivots[i]
      CK(cudaEventRecord(ctx->ev_piv, s));
      CK(cudaStreamWaitEvent(ctx->side, ctx->ev_piv, 0));
      const uint32_t* xl = ctx->det_from_cur ? ctx->cur_limbs : ctx->det_limbs + (i - 1);
      int64_t xc = ctx->det_from_cur ? 1 : n;
      const int32_t* xe = ctx->det_from_cur ? ctx->cur_exp : ctx->det_exp + (i - 1);
      const uint8_t* xk = ctx->det_from_cur ? ctx->cur_cls : ctx->det_cls + (i - 1);
      int rc = mul_row_launch(&ctx->plan, ctx->side, xl, xc, xe, xk, ctx->piv_limbs + i, n, ctx->piv_exp + i,
                              ctx->piv_cls + i, 1, ctx->det_limbs + i, n, ctx->det_exp + i, ctx->det_cls + i,
                              ctx->status, &ctx->launches, i, ctx->ws_dx, ctx->ws_dy);
      if (rc != DS_OK) { ctx->err = "det product launch failed"; return rc; }
    }
  } else {
    k_pivot<<<1, 32, 0, s>>>(k, i);
    ctx->launches++;
  }
  ctx->host_have_det = 1;
  ctx->det_from_cur = 0;
  int jl0 = first_local_after(i, ctx->rank, ctx->world, ctx->row_base);
  int nrows = ctx->nloc - jl0;
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (ctx->prof_on && nrows > 0) {
    if (ctx->prof_used + 2 > ctx->prof_ev.size()) {
      for (int q = 0; q < 256; q++) {
        cudaEvent_t ev;
        CK(cudaEventCreate(&ev));
        ctx->prof_ev.push_back(ev);
      }
    }
    pe0 = ctx->prof_ev[ctx->prof_used];
    pe1 = ctx->prof_ev[ctx->prof_used + 1];
    ctx->prof_used += 2;
  }
  if (nrows > 0) {
    // ---- multipliers z_j = RN(a_ji / piv), a_ji <- -z_j (elim.py:47, 53)
    if (fast && la_have) {
      CK(cudaStreamWaitEvent(s, ctx->ev_mult, 0));  // computed by the previous step's lookahead
    } else if (fast && wdiv_ok(ctx)) {
      int blocks = (nrows + wpb - 1) / wpb;
      size_t smem = (size_t)wpb * wwords * 4;
      WDIV_DISPATCH(K, k_mult_w, blocks, 32 * wpb, smem, s, k, i, jl0, wwords, 0, nullptr);
    } else if (cxf) {
      int cw_words = 0;
      const int cw_wpb = cw_plan(ctx, &cw_words);
      if (cw_wpb >= 1) {  // one warp per (row, component)
        const unsigned nb = (unsigned)((2 * (int64_t)nrows + cw_wpb - 1) / cw_wpb);
        k_cw_mult<<<nb, 32 * cw_wpb, (size_t)cw_wpb * cw_words * 4, s>>>(k, i, jl0, cw_words);
      } else {
        KArgs km = k;
        const size_t sm = cx_smem_launch(ctx, &km, 2 * (int64_t)nrows);
        if (km.sm_threads)
          k_mult_c2<<<(unsigned)((2 * (int64_t)nrows + km.sm_threads - 1) / km.sm_threads), km.sm_threads, sm, s>>>(
              km, i, jl0);
        else
          k_mult_c2<<<grid_for(ctx, 2 * (int64_t)nrows, 64), 64, 0, s>>>(k, i, jl0);
      }
      k_neg_z<<<grid_for(ctx, 2 * (int64_t)nrows, 64), 64, 0, s>>>(k, i, jl0);
      ctx->launches++;
    } else {
      k_mult<<<grid_for(ctx, nrows, 64), 64, 0, s>>>(k, i, jl0);
    }
    ctx->launches++;
    // ---- update of the trailing rows (elim.py:49-52)
    int ncols_u = collect_minors ? n - 1 : n - 1 - i;
    if (pe0) {
      CK(cudaEventRecord(pe0, s));
      ctx->prof_launches++;
      ctx->prof_work += (double)nrows * ncols_u * (double)L * L * (ctx->kind == DS_KIND_COMPLEX ? 4.0 : 1.0);
    }
    if (fast) {
      // lookahead for step i + 1 (one rank, inside the current ds_run range, rows left)
      const int la_col = (ctx->tc.enabled && ((ctx->world == 1 && ctx->row_base == 0) || ctx->la_ext) &&
                          i + 1 < ctx->la_limit &&
                          i + 2 < n && !getenv("DS_NO_LOOKAHEAD"))
                             ? i + 1
                             : -1;
      int la_used = 0;
      int rc = ctx->tc.enabled
                   ? tc_update_launch(&ctx->tc, s, ctx->a_limbs, ctx->a_exp, ctx->a_cls, ctx->a_count, ctx->pbuf,
                                      ctx->z_limbs, ctx->z_exp, ctx->z_cls, ctx->nloc, n, i, jl0, collect_minors,
                                      ctx->status, &ctx->launches, ctx->la, ctx->ev_prep, ctx->ev_a, la_col, &la_used)
                   : update_launch(&ctx->plan, s, ctx->a_limbs, ctx->a_exp, ctx->a_cls, ctx->a_count, ctx->pbuf,
                                   ctx->z_limbs, ctx->z_exp, ctx->z_cls, ctx->nloc, n, i, jl0, collect_minors,
                                   ctx->status, &ctx->launches);
      if (rc != DS_OK) {
        ctx->err = g_last_error.empty() ? std::string("update launch: ") + cudaGetErrorString(cudaGetLastError())
                                        : g_last_error;
        return rc;
      }
      if (ctx->la_ext) {
        // caller-driven lookahead: it stages / broadcasts a_{i+1,i+1} and launches
        // the multipliers (ds_lookahead_pivot, ds_lookahead_mult) on the lookahead
        // stream; without the tile split that stream must see the whole update
        if (!la_used) {
          CK(cudaEventRecord(ctx->ev_a, s));
          CK(cudaStreamWaitEvent(ctx->la, ctx->ev_a, 0));
        }
      } else if (la_used) {
        // column i+1 is final: step i+1's multipliers on the lookahead stream (after
        // the tile holding that column) while the other tiles of step i still run
        KArgs kn = k;
        kn.z_limbs = ctx->zb_limbs[(i + 1) & 1];
        kn.z_exp = ctx->zb_exp[(i + 1) & 1];
        kn.z_cls = ctx->zb_cls[(i + 1) & 1];
        const int jl1 = i + 2;  // world 1: local row = global row
        const int rows1 = ctx->nloc - jl1;
        int blocks = (rows1 + wpb - 1) / wpb;
        size_t smem = (size_t)wpb * wwords * 4;
        WDIV_DISPATCH(K, k_mult_w, blocks, 32 * wpb, smem, ctx->la, kn, i + 1, jl1, wwords, 1, nullptr);
        ctx->launches++;
        CK(cudaEventRecord(ctx->ev_mult, ctx->la));
        ctx->la_step = i + 1;
      }
    } else if (ctx->kind == DS_KIND_COMPLEX && ctx->tc.enabled && !force_general()) {
      // complex: the four component products on the wide tensor-core engine
      int rc = tc_update_launch(&ctx->tc, s, ctx->a_limbs, ctx->a_exp, ctx->a_cls, ctx->a_count, ctx->pbuf,
                                ctx->z_limbs, ctx->z_exp, ctx->z_cls, ctx->nloc, n, i, jl0, collect_minors,
                                ctx->status, &ctx->launches);
      if (rc != DS_OK) { ctx->err = g_last_error; return rc; }
    } else {
      int kfirst = collect_minors ? 0 : i + 1;
      int64_t ncols = n - kfirst - (collect_minors ? 1 : 0);
      if (ncols > 0) {
        k_update_general<<<grid_for(ctx, nrows * ncols, 128), 128, 0, s>>>(k, i, jl0, collect_minors);
        ctx->launches++;
      }
    }
    if (pe1) CK(cudaEventRecord(pe1, s));
  }
  // ---- minors of leading size m = i+2 (elim.py:220-226)
  if (collect_minors && i + 1 < n) {
    int m = i + 2;
    if ((series || m == n) && owns_row(ctx, i + 1)) {
      int mrc = ensure_minors(ctx);
      if (mrc != DS_OK) return mrc;
      k = kargs(ctx);  // minors pointers
      ks = k;
      ks.scratch = ctx->scratch_side;
      int64_t jl = (i + 1 - ctx->row_base) / ctx->world;
      if (fast) {
        // outputs only: run on the side stream after this step's update
        cudaStream_t ss = ctx->side;
        CK(cudaEventRecord(ctx->ev_upd, s));
        CK(cudaStreamWaitEvent(ss, ctx->ev_upd, 0));
        const int64_t mo = (jl % ctx->m_rows) * n;
        int rc = mul_row_launch(&ctx->plan, ss, ctx->det_limbs + i, n, ctx->det_exp + i, ctx->det_cls + i,
                                ctx->a_limbs + jl * n, ctx->a_count, ctx->a_exp + jl * n, ctx->a_cls + jl * n, i + 1,
                                ctx->sig_limbs + mo, ctx->m_count, ctx->sig_exp + mo, ctx->sig_cls + mo,
                                ctx->status, &ctx->launches, i, ctx->ws_ex, ctx->ws_ey);
        if (rc != DS_OK) { ctx->err = "minor product launch failed"; return rc; }
        k_emit_last<<<1, 128, 0, ss>>>(k, i);
        if (wdiv_ok(ctx)) {
          int blocks = (m + wpb - 1) / wpb;
          size_t smem = (size_t)wpb * wwords * 4;
          WDIV_DISPATCH(K, k_emit_norm_w, blocks, 32 * wpb, smem, ss, k, i, wwords);
        } else {
          k_emit_norm<<<grid_for(ctx, m, 64), 64, 0, ss>>>(k, i);
        }
        ctx->launches += 2;
      } else if (cxf) {
        cudaStream_t ss = ctx->side;
        CK(cudaEventRecord(ctx->ev_upd, s));
        CK(cudaStreamWaitEvent(ss, ctx->ev_upd, 0));
        int cw_words = 0;
        const int cw_wpb = cw_plan(ctx, &cw_words);
        KArgs ke = ks;
        const size_t sm = cw_wpb >= 1 ? 0 : cx_smem_launch(ctx, &ke, 2 * (int64_t)m);
        if (cw_wpb >= 1) {  // one warp per (entry, component)
          const unsigned nb = (unsigned)((2 * (int64_t)m + cw_wpb - 1) / cw_wpb);
          const size_t smw = (size_t)cw_wpb * cw_words * 4;
          k_cw_emit_signed<<<nb, 32 * cw_wpb, smw, ss>>>(ks, i, cw_words);
          k_cw_emit_norm<<<nb, 32 * cw_wpb, smw, ss>>>(ks, i, cw_words);
        } else if (ke.sm_threads) {
          const unsigned nb = (unsigned)((2 * (int64_t)m + ke.sm_threads - 1) / ke.sm_threads);
          k_emit_signed_c2<<<nb, ke.sm_threads, sm, ss>>>(ke, i);
          k_emit_norm_c2<<<nb, ke.sm_threads, sm, ss>>>(ke, i);
        } else {
          k_emit_signed_c2<<<grid_for(ctx, 2 * (int64_t)m, 64), 64, 0, ss>>>(ks, i);
          k_emit_norm_c2<<<grid_for(ctx, 2 * (int64_t)m, 64), 64, 0, ss>>>(ks, i);
        }
        ctx->launches += 2;
      } else {
        k_emit_signed<<<grid_for(ctx, m, 64), 64, 0, s>>>(k, i);
        k_emit_norm<<<grid_for(ctx, m, 64), 64, 0, s>>>(k, i);
        ctx->launches += 2;
      }
    }
  }
  CK(cudaGetLastError());
  return DS_OK;
}

int ds_snapshot(ds_ctx* ctx, int save) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->side));
  int nc = ctx->ncomp, L = ctx->L;
  size_t lb = sizeof(uint32_t) * nc * L * ctx->a_count, eb = sizeof(int32_t) * nc * ctx->a_count,
         cb = (size_t)nc * ctx->a_count;
  if (save) {
    int rc;
    if (!ctx->snap_limbs) {
      if ((rc = dmalloc(ctx, &ctx->snap_limbs, lb / 4)) != DS_OK) return rc;
      if ((rc = dmalloc(ctx, &ctx->snap_exp, eb / 4)) != DS_OK) return rc;
      if ((rc = dmalloc(ctx, &ctx->snap_cls, cb)) != DS_OK) return rc;
    }
    CK(cudaMemcpyAsync(ctx->snap_limbs, ctx->a_limbs, lb, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->snap_exp, ctx->a_exp, eb, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->snap_cls, ctx->a_cls, cb, cudaMemcpyDeviceToDevice, ctx->stream));
    return DS_OK;
  }
  if (!ctx->snap_limbs) return DS_INVALID;
  CK(cudaMemcpyAsync(ctx->a_limbs, ctx->snap_limbs, lb, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->a_exp, ctx->snap_exp, eb, cudaMemcpyDeviceToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->a_cls, ctx->snap_cls, cb, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->host_have_det = 0;
  ctx->la_step = -1;
  ctx->det_from_cur = 0;
  CK(cudaMemsetAsync(ctx->row_flags, 0, ctx->n, ctx->stream));
  if (ctx->swaps) CK(cudaMemsetAsync(ctx->swaps, 0, ctx->n, ctx->stream));
  CK(cudaMemsetAsync(ctx->status + 1, 0, 7 * sizeof(int32_t), ctx->stream));
  CK(cudaMemsetAsync(ctx->status, 0xff, sizeof(int32_t), ctx->stream));  // -1
  ctx->st_next = 1;
  ctx->st_pending = 0;
  return DS_OK;
}

int ds_profile(ds_ctx* ctx, int enable) {
  ctx->prof_on = enable ? 1 : 0;
  return DS_OK;
}

int ds_profile_read(ds_ctx* ctx, double* ms, int64_t* launches, double* work) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  double tot = 0;
  for (size_t q = 0; q + 1 < ctx->prof_used; q += 2) {
    float f = 0;
    CK(cudaEventElapsedTime(&f, ctx->prof_ev[q], ctx->prof_ev[q + 1]));
    tot += f;
  }
  *ms = tot;
  *launches = ctx->prof_launches;
  *work = ctx->prof_work;
  ctx->prof_used = 0;
  ctx->prof_launches = 0;
  ctx->prof_work = 0;
  return DS_OK;
}

int ds_lookahead_enable(ds_ctx* ctx, int limit) {
  if (ctx->row_base != 0 && limit > 0) return DS_INVALID;
  if (limit > 0 && (!fast_real(ctx) || !wdiv_ok(ctx))) return DS_INVALID;  // needs the warp division
  ctx->la_limit = limit;
  ctx->la_ext = limit > 0 ? 1 : 0;
  if (limit <= 0) ctx->la_step = -1;
  return DS_OK;
}

int ds_lookahead_stream(ds_ctx* ctx, void** stream) {
  *stream = (void*)ctx->la;
  return DS_OK;
}

int ds_lookahead_pivot(ds_ctx* ctx, int i1, void* buf) {
  if (i1 < 0 || i1 >= ctx->n || i1 % ctx->world != ctx->rank || !fast_real(ctx)) return DS_INVALID;
  CK(cudaSetDevice(ctx->device));
  KArgs k = kargs(ctx);
  k_pscal_stage<<<1, 128, 0, ctx->la>>>(k, i1, (int64_t)(i1 / ctx->world), (uint8_t*)buf);
  ctx->launches++;
  CK(cudaGetLastError());
  return DS_OK;
}

int ds_lookahead_mult(ds_ctx* ctx, int i1, const void* buf) {
  if (i1 < 0 || i1 >= ctx->n || !fast_real(ctx) || !wdiv_ok(ctx)) return DS_INVALID;
  CK(cudaSetDevice(ctx->device));
  KArgs k = kargs(ctx);
  k.z_limbs = ctx->zb_limbs[i1 & 1];
  k.z_exp = ctx->zb_exp[i1 & 1];
  k.z_cls = ctx->zb_cls[i1 & 1];
  const int L = ctx->L;
  const int K = warp_k(L);
  const int wwords = wdiv_words(L, ctx->p, K);
  const int wpb = 4;
  int maxsm = 0;
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  set_wdiv_attrs(maxsm);
  const int jl1 = first_local_after(i1, ctx->rank, ctx->world);
  const int rows1 = ctx->nloc - jl1;
  if (rows1 > 0) {
    int blocks = (rows1 + wpb - 1) / wpb;
    size_t smem = (size_t)wpb * wwords * 4;
    WDIV_DISPATCH(K, k_mult_w, blocks, 32 * wpb, smem, ctx->la, k, i1, jl1, wwords, 0, (const uint8_t*)buf);
    ctx->launches++;
  }
  CK(cudaEventRecord(ctx->ev_mult, ctx->la));
  ctx->la_step = i1;
  CK(cudaGetLastError());
  return DS_OK;
}

int ds_counters(ds_ctx* ctx, int64_t* out, int n) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->side));
  int32_t st[8];
  CK(cudaMemcpyAsync(st, ctx->status, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int64_t v[6] = {(int64_t)(uint32_t)st[6], ctx->tc.enabled ? 1 : 0, (ctx->plan.fused && !ctx->tc.enabled) ? 1 : 0,
                  (int64_t)(uint32_t)st[7], ctx->h2d_bytes, ctx->d2h_bytes};
  for (int q = 0; q < n && q < 6; q++) out[q] = v[q];
  return DS_OK;
}

int ds_status(ds_ctx* ctx, int* failed_step) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->side));
  int32_t st[8];
  CK(cudaMemcpyAsync(st, ctx->status, sizeof(st), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *failed_step = st[0];
  if (st[2] != 0) {
    ctx->err = "exponent left the MPFR default range";
    return DS_OVERFLOW;
  }
  if (st[4] != 0 || st[5] != 0) {  // internal consistency counters: must stay zero
    ctx->err = st[4] ? "update engine: normalisation misprediction" : "tensor-core update: fallback list overflow";
    return DS_CUDA;
  }
  return DS_OK;
}

int ds_set_det(ds_ctx* ctx, const ds_soa* d) {
  CK(cudaSetDevice(ctx->device));
  int L = ctx->L;
  for (int c = 0; c < ctx->ncomp; c++) {
    for (int l = 0; l < L; l++)
      CK(cudaMemcpyAsync(ctx->cur_limbs + (int64_t)c * L + l, d->limbs + ((int64_t)c * L + l) * d->count,
                         sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->cur_exp + c, d->exp + (int64_t)c * d->count, sizeof(int32_t), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(ctx->cur_cls + c, d->cls + (int64_t)c * d->count, 1, cudaMemcpyHostToDevice, ctx->stream));
  }
  int one = 1;
  CK(cudaMemcpyAsync(ctx->status + 1, &one, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  ctx->host_have_det = 1;
  ctx->det_from_cur = 1;
  CK(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

static int copy_vec(ds_ctx* ctx, ds_soa* dst, const uint32_t* limbs, const int32_t* ex, const uint8_t* cl,
                    int64_t src_count, int64_t n_items) {
  if (!dst || !dst->limbs || n_items <= 0) return DS_OK;
  int L = ctx->L;
  ctx->d2h_bytes += (int64_t)ctx->ncomp * (4 * L + 5) * n_items;
  for (int c = 0; c < ctx->ncomp; c++) {
    for (int l = 0; l < L; l++)
      CK(cudaMemcpyAsync(dst->limbs + ((int64_t)c * L + l) * dst->count, limbs + ((int64_t)c * L + l) * src_count,
                         sizeof(uint32_t) * n_items, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(dst->exp + (int64_t)c * dst->count, ex + (int64_t)c * src_count, sizeof(int32_t) * n_items,
                       cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(dst->cls + (int64_t)c * dst->count, cl + (int64_t)c * src_count, n_items,
                       cudaMemcpyDeviceToHost, ctx->stream));
  }
  return DS_OK;
}

// minors rows [r0, r1) of a world-1 context, the first `width` entries of each
// (row m-1 holds m entries), on stream s: one 2D copy per limb plane
// local minors rows [r0, r1) (ring slots r % m_rows; split where the ring wraps)
// into host rows starting at hrow0 (row pitch n) of dst
static int copy_row_range_to(ds_ctx* ctx, ds_soa* dst, const uint32_t* limbs, const int32_t* ex, const uint8_t* cl,
                             int r0, int r1, int width, cudaStream_t s, int hrow0) {
  if (!dst || !dst->limbs || r1 <= r0 || width <= 0) return DS_OK;
  if (!limbs) return DS_OK;  // nothing emitted yet
  const int n = ctx->n, L = ctx->L;
  ctx->d2h_bytes += (int64_t)ctx->ncomp * (4 * L + 5) * (int64_t)(r1 - r0) * width;
  for (int a = r0; a < r1;) {
    const int slot = a % ctx->m_rows;
    const int b = std::min(r1, a + (ctx->m_rows - slot));
    const size_t rows = (size_t)(b - a);
    const int64_t o = (int64_t)slot * n, ho = (int64_t)(hrow0 + (a - r0)) * n;
    for (int c = 0; c < ctx->ncomp; c++) {
      for (int l = 0; l < L; l++)
        CK(cudaMemcpy2DAsync(dst->limbs + ((int64_t)c * L + l) * dst->count + ho, sizeof(uint32_t) * n,
                             limbs + ((int64_t)c * L + l) * ctx->m_count + o, sizeof(uint32_t) * n,
                             sizeof(uint32_t) * width, rows, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpy2DAsync(dst->exp + (int64_t)c * dst->count + ho, sizeof(int32_t) * n,
                           ex + (int64_t)c * ctx->m_count + o, sizeof(int32_t) * n, sizeof(int32_t) * width, rows,
                           cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpy2DAsync(dst->cls + (int64_t)c * dst->count + ho, n, cl + (int64_t)c * ctx->m_count + o, n, width,
                           rows, cudaMemcpyDeviceToHost, s));
    }
    a = b;
  }
  return DS_OK;
}

static int copy_row_range(ds_ctx* ctx, ds_soa* dst, const uint32_t* limbs, const int32_t* ex, const uint8_t* cl,
                          int r0, int r1, int width, cudaStream_t s) {
  return copy_row_range_to(ctx, dst, limbs, ex, cl, r0, r1, width, s, r0);
}

static bool host_pinned(const void* p) {
  cudaPointerAttributes at;
  if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

static int copy_rows(ds_ctx* ctx, ds_soa* dst, const uint32_t* limbs, const int32_t* ex, const uint8_t* cl) {
  // owned minors rows (local index jl <-> global row rank + jl*world) into a
  // full n*n host matrix
  if (!dst || !dst->limbs || !limbs) return DS_OK;
  if (ctx->m_rows < ctx->nloc) {
    ctx->err = "minors are streamed (ds_stream_minors): they are not resident for a full fetch";
    return DS_INVALID;
  }
  int n = ctx->n, L = ctx->L;
  int64_t r0, rs;
  if (!host_rows(ctx, dst->count, &r0, &rs)) return DS_INVALID;
  for (int c = 0; c < ctx->ncomp; c++) {
    for (int l = 0; l < L; l++)
      CK(cudaMemcpy2DAsync(dst->limbs + ((int64_t)c * L + l) * dst->count + r0 * n,
                           sizeof(uint32_t) * n * rs, limbs + ((int64_t)c * L + l) * ctx->m_count,
                           sizeof(uint32_t) * n, sizeof(uint32_t) * n, ctx->nloc, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpy2DAsync(dst->exp + (int64_t)c * dst->count + r0 * n, sizeof(int32_t) * n * rs,
                         ex + (int64_t)c * ctx->m_count, sizeof(int32_t) * n, sizeof(int32_t) * n, ctx->nloc,
                         cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpy2DAsync(dst->cls + (int64_t)c * dst->count + r0 * n, (size_t)n * rs,
                         cl + (int64_t)c * ctx->m_count, n, n, ctx->nloc, cudaMemcpyDeviceToHost, ctx->stream));
  }
  ctx->d2h_bytes += (int64_t)ctx->ncomp * (4 * L + 5) * ctx->nloc * n;
  return DS_OK;
}

// minors_from: minors rows below it were already copied (progressive D2H in ds_run)
static int results_fetch_from(ds_ctx* ctx, int upto, ds_results* r, int minors_from) {
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->side));
  int rc;
  if ((rc = copy_vec(ctx, &r->pivots, ctx->piv_limbs, ctx->piv_exp, ctx->piv_cls, ctx->n, upto)) != DS_OK) return rc;
  if ((rc = copy_vec(ctx, &r->dets, ctx->det_limbs, ctx->det_exp, ctx->det_cls, ctx->n, upto)) != DS_OK) return rc;
  if (minors_from > 0) {
    if ((rc = copy_row_range(ctx, &r->signed_minors, ctx->sig_limbs, ctx->sig_exp, ctx->sig_cls, minors_from, ctx->n,
                             ctx->n, ctx->stream)) != DS_OK)
      return rc;
    if ((rc = copy_row_range(ctx, &r->normalized, ctx->nrm_limbs, ctx->nrm_exp, ctx->nrm_cls, minors_from, ctx->n,
                             ctx->n, ctx->stream)) != DS_OK)
      return rc;
  } else {
    if ((rc = copy_rows(ctx, &r->signed_minors, ctx->sig_limbs, ctx->sig_exp, ctx->sig_cls)) != DS_OK) return rc;
    if ((rc = copy_rows(ctx, &r->normalized, ctx->nrm_limbs, ctx->nrm_exp, ctx->nrm_cls)) != DS_OK) return rc;
  }
  if (r->row_flags) {
    // flags of rows this rank owns (m-1 % world == rank)
    uint8_t* tmp = (uint8_t*)malloc(ctx->n);
    CK(cudaMemcpyAsync(tmp, ctx->row_flags, ctx->n, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->d2h_bytes += ctx->n;
    CK(cudaStreamSynchronize(ctx->stream));
    for (int jl = 0; jl < ctx->nloc; jl++) {
      const int m1 = ctx->row_base + ctx->rank + jl * ctx->world;
      if (m1 < ctx->n) r->row_flags[m1] = tmp[m1];
    }
    free(tmp);
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_results_fetch(ds_ctx* ctx, int upto, ds_results* r) { return results_fetch_from(ctx, upto, r, 0); }

// trace entries [t0, t1) and minors rows of leading sizes [m0, m1) (row m-1,
// its first m entries) with their flags: the incremental fetch the drop-in
// eliminate() streams rows to its sink with (world 1)
int ds_results_fetch_range(ds_ctx* ctx, int t0, int t1, int m0, int m1, ds_results* r) {
  if (ctx->world != 1 || ctx->row_base != 0) return DS_INVALID;
  if (t0 < 0 || t1 > ctx->n || m0 < 2 || m1 > ctx->n + 1) return DS_INVALID;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->side));
  CK(cudaStreamSynchronize(ctx->stream));
  const int n = ctx->n, L = ctx->L;
  if (t1 > t0) {
    const int64_t cnt = t1 - t0;
    ds_soa* vs[2] = {&r->pivots, &r->dets};
    uint32_t* sl[2] = {ctx->piv_limbs, ctx->det_limbs};
    int32_t* se[2] = {ctx->piv_exp, ctx->det_exp};
    uint8_t* sc[2] = {ctx->piv_cls, ctx->det_cls};
    for (int v = 0; v < 2; v++) {
      ds_soa* d = vs[v];
      if (!d->limbs) continue;
      ctx->d2h_bytes += (int64_t)ctx->ncomp * (4 * L + 5) * cnt;
      for (int c = 0; c < ctx->ncomp; c++) {
        for (int l = 0; l < L; l++)
          CK(cudaMemcpyAsync(d->limbs + ((int64_t)c * L + l) * d->count + t0, sl[v] + ((int64_t)c * L + l) * n + t0,
                             sizeof(uint32_t) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(d->exp + (int64_t)c * d->count + t0, se[v] + (int64_t)c * n + t0, sizeof(int32_t) * cnt,
                           cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(d->cls + (int64_t)c * d->count + t0, sc[v] + (int64_t)c * n + t0, cnt,
                           cudaMemcpyDeviceToHost, ctx->stream));
      }
    }
  }
  if (m1 > m0) {
    int rc;
    if ((rc = copy_row_range(ctx, &r->signed_minors, ctx->sig_limbs, ctx->sig_exp, ctx->sig_cls, m0 - 1, m1 - 1, m1 - 1,
                             ctx->stream)) != DS_OK)
      return rc;
    if ((rc = copy_row_range(ctx, &r->normalized, ctx->nrm_limbs, ctx->nrm_exp, ctx->nrm_cls, m0 - 1, m1 - 1, m1 - 1,
                             ctx->stream)) != DS_OK)
      return rc;
    if (r->row_flags) {
      CK(cudaMemcpyAsync(r->row_flags + (m0 - 1), ctx->row_flags + (m0 - 1), (size_t)(m1 - m0),
                         cudaMemcpyDeviceToHost, ctx->stream));
      ctx->d2h_bytes += m1 - m0;
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return DS_OK;
}

int ds_set_pivot_mode(ds_ctx* ctx, int mode) {
  if (mode != 0 && mode != 1) return DS_INVALID;
  if (mode == 1 && (ctx->world != 1 || ctx->row_base != 0 || ctx->kind != DS_KIND_REAL)) {
    ctx->err = "pivot_mode='partial' runs on the serial real engine only (world 1, kind real)";
    return DS_INVALID;
  }
  CK(cudaSetDevice(ctx->device));
  if (mode == 1 && !ctx->swaps) {
    int rc;
    if ((rc = dmalloc(ctx, &ctx->swaps, (size_t)ctx->n)) != DS_OK) return rc;
    if ((rc = dmalloc(ctx, &ctx->pbest, 1)) != DS_OK) return rc;
    CK(cudaMemsetAsync(ctx->swaps, 0, ctx->n, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  ctx->pivot_partial = mode;
  return DS_OK;
}

int ds_swaps_fetch(ds_ctx* ctx, int upto_step, uint8_t* swapped) {
  if (upto_step < 0 || upto_step > ctx->n) return DS_INVALID;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  if (!ctx->swaps) {
    memset(swapped, 0, (size_t)upto_step);
    return DS_OK;
  }
  CK(cudaMemcpy(swapped, ctx->swaps, (size_t)upto_step, cudaMemcpyDeviceToHost));
  return DS_OK;
}

int ds_run(ds_ctx* ctx, int collect_minors, int series, int start_step, int stop_step, ds_results* res,
           int* steps_done) {
  if (ctx->world != 1 || ctx->row_base != 0) return DS_INVALID;
  if (start_step < 0 || stop_step > ctx->n || start_step > stop_step) return DS_INVALID;
  if (ctx->pivot_partial && collect_minors) {  // elim.py:186-187
    ctx->err = "partial pivoting cannot be combined with minors collection";
    return DS_INVALID;
  }
  int rc;
  // progressive D2H of the minors (pinned host buffers): rows finalised by
  // the emission are copied in batches on the side stream while the
  // elimination runs -- row m-1 holds m entries (triangle)
  const bool streaming = ctx->st_batch > 0 && collect_minors;
  if (streaming && start_step + 1 > ctx->st_next) ctx->st_next = start_step + 1;
  const bool prog = !streaming && res && collect_minors && series && res->signed_minors.limbs && res->normalized.limbs &&
                    host_pinned(res->signed_minors.limbs) && host_pinned(res->normalized.limbs) &&
                    host_pinned(res->signed_minors.exp) && host_pinned(res->signed_minors.cls) &&
                    host_pinned(res->normalized.exp) && host_pinned(res->normalized.cls) &&
                    res->signed_minors.count == (int64_t)ctx->n * ctx->n && !getenv("DS_NO_PROGRESSIVE_D2H");
  const int BATCH = 64;
  int copied = 0;
  ctx->la_ext = 0;  // single-rank run: the engine chains the lookahead itself
  // row swaps change column i+1's owner rows after the update: no lookahead
  ctx->la_limit = ctx->pivot_partial ? -1 : stop_step;
  for (int i = start_step; i < stop_step; i++) {
    if (ctx->pivot_partial) {
      KArgs k = kargs(ctx);
      k_pivot_select<<<1, 1024, 0, ctx->stream>>>(k, i, ctx->pbest, ctx->swaps);
      k_swap_rows<<<grid_for(ctx, (int64_t)ctx->ncomp * (ctx->L + 2) * ctx->n, 256), 256, 0, ctx->stream>>>(
          k, i, ctx->pbest);
      ctx->launches += 2;
      CK(cudaGetLastError());
    }
    if ((rc = ds_pivot_stage(ctx, i)) != DS_OK) { ctx->la_limit = -1; return rc; }
    if ((rc = ds_step(ctx, i, collect_minors, series)) != DS_OK) { ctx->la_limit = -1; return rc; }
    if (streaming && (i + 1 - start_step) % ctx->st_batch == 0 &&
        (rc = ds_stream_flush(ctx, i + 1, 0)) != DS_OK) {
      ctx->la_limit = -1;
      return rc;
    }
    if (prog && (i + 1 - start_step) % BATCH == 0) {
      const int r1 = i + 2 < ctx->n ? i + 2 : ctx->n;  // rows 0 .. i+1 are final after step i
      if ((rc = copy_row_range(ctx, &res->signed_minors, ctx->sig_limbs, ctx->sig_exp, ctx->sig_cls, copied, r1, r1,
                               ctx->side)) != DS_OK ||
          (rc = copy_row_range(ctx, &res->normalized, ctx->nrm_limbs, ctx->nrm_exp, ctx->nrm_cls, copied, r1, r1,
                               ctx->side)) != DS_OK) {
        ctx->la_limit = -1;
        return rc;
      }
      copied = r1;
    }
  }
  ctx->la_limit = -1;
  ctx->la_step = -1;
  CK(cudaEventRecord(ctx->ev_la_done, ctx->la));  // nothing of the lookahead stream is left behind
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_la_done, 0));
  int failed;
  rc = ds_status(ctx, &failed);
  int upto = failed >= 0 ? failed : stop_step;
  *steps_done = upto;
  if (streaming) {
    int rc2 = ds_stream_flush(ctx, upto, 1);
    if (rc2 != DS_OK) return rc2;
  }
  if (res) {
    int rc2 = results_fetch_from(ctx, upto, res, streaming ? ctx->n : (prog ? copied : 0));
    if (rc2 != DS_OK) return rc2;
  }
  if (rc != DS_OK) return rc;
  return failed >= 0 ? DS_ZERO_PIVOT : DS_OK;
}

int ds_scalar_op(int op, int kind, long prec_bits, int device, const ds_soa* a, const ds_soa* b, ds_soa* out) {
  ds_ctx* ctx = nullptr;
  if (prec_bits < 64 || a->count != b->count || a->count != out->count) return DS_INVALID;
  CK(cudaSetDevice(device));
  int L = nlimbs(prec_bits), nc = kind == DS_KIND_COMPLEX ? 2 : 1;
  int64_t cnt = a->count;
  if (cnt == 0) return DS_OK;
  size_t lb = sizeof(uint32_t) * nc * L * cnt, eb = sizeof(int32_t) * nc * cnt, cb = (size_t)nc * cnt;
  uint8_t* buf;
  int64_t sthreads = 148 * 4 * 128;
  int64_t swords = general_scratch_words(L, kind);
  size_t total = 3 * (lb + eb + cb) + 64 + sizeof(uint32_t) * sthreads * swords + 64;
  CK(cudaMalloc(&buf, total));
  uint8_t* q = buf;
  auto take = [&](size_t bytes) { uint8_t* r = q; q += (bytes + 15) & ~(size_t)15; return r; };
  uint32_t *al = (uint32_t*)take(lb), *bl = (uint32_t*)take(lb), *ol = (uint32_t*)take(lb);
  int32_t *ae = (int32_t*)take(eb), *be = (int32_t*)take(eb), *oe = (int32_t*)take(eb);
  uint8_t *ac = take(cb), *bc = take(cb), *oc = take(cb);
  int32_t* st = (int32_t*)take(64);
  uint32_t* scratch = (uint32_t*)take(sizeof(uint32_t) * sthreads * swords);
  CK(cudaMemcpy(al, a->limbs, lb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(bl, b->limbs, lb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ae, a->exp, eb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(be, b->exp, eb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ac, a->cls, cb, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(bc, b->cls, cb, cudaMemcpyHostToDevice));
  CK(cudaMemset(st, 0, 64));
  int block = 128;
  int64_t g = (cnt + block - 1) / block;
  if (g > sthreads / block) g = sthreads / block;
  k_scalar_op<<<(int)g, block>>>(op, kind, L, (int)prec_bits, cnt, al, ae, ac, bl, be, bc, ol, oe, oc, scratch,
                                 sthreads, st);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out->limbs, ol, lb, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out->exp, oe, eb, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(out->cls, oc, cb, cudaMemcpyDeviceToHost));
  int32_t hst[16];
  CK(cudaMemcpy(hst, st, 64, cudaMemcpyDeviceToHost));
  CK(cudaFree(buf));
  return hst[2] ? DS_OVERFLOW : DS_OK;
}

}  // extern "C"
