// api.cu — the C ABI (include/mbci.h): validation, plan selection, TMA descriptor encoding,
// launches, end-to-end host entry, and the selector's host-only entry points.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mbci.h"
#include "chain_tc6.cuh"   // kT5Threads, kT6Threads (the kernels are instantiated in k_*.cu)
#include "kernels.h"
#include "search.h"
#include "selector.h"

using namespace mbci;

namespace {

thread_local std::string g_err;

mbci_status_t fail(mbci_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

mbci_status_t cuda_fail(cudaError_t e, const char* what) {
  return fail(MBCI_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// Validate and fill packed strides.
mbci_status_t normalize(const mbci_chain_desc_t* in, mbci_chain_desc_t* d) {
  if (!in) return fail(MBCI_ERR_INVALID, "desc is NULL");
  *d = *in;
  if (d->batch < 0 || d->M < 0 || d->N < 0 || d->K < 0 || d->L < 0)
    return fail(MBCI_ERR_INVALID, "negative dimension");
  if (d->dtype < MBCI_F32 || d->dtype > MBCI_BF16) return fail(MBCI_ERR_INVALID, "bad dtype %d", d->dtype);
  if (d->op < MBCI_OP_NONE || d->op > MBCI_OP_GELU) return fail(MBCI_ERR_INVALID, "bad op %d", d->op);
  if (d->mask < MBCI_MASK_NONE || d->mask > MBCI_MASK_CAUSAL_KEY_PADDING)
    return fail(MBCI_ERR_INVALID, "bad mask %d", d->mask);
  if (d->mask != MBCI_MASK_NONE && d->op != MBCI_OP_SOFTMAX)
    return fail(MBCI_ERR_INVALID, "masks require op SOFTMAX");
  if (d->b_layout != 0 && d->b_layout != 1) return fail(MBCI_ERR_INVALID, "bad b_layout %d", d->b_layout);
  if (d->tune < 0 || d->tune > 2) return fail(MBCI_ERR_INVALID, "bad tune %d", d->tune);
  if (d->K > kMaxK || d->L > kMaxL)
    return fail(MBCI_ERR_UNSUPPORTED, "K=%lld L=%lld: this build takes K, L <= %lld",
                (long long)d->K, (long long)d->L, (long long)kMaxK);
  const int64_t b_inner = d->b_layout == 0 ? d->N : d->K;
  const int64_t b_rows = d->b_layout == 0 ? d->K : d->N;
  if (d->ld_a == 0) d->ld_a = d->K;
  if (d->ld_b == 0) d->ld_b = b_inner;
  if (d->ld_d == 0) d->ld_d = d->L;
  if (d->ld_e == 0) d->ld_e = d->L;
  if (d->bs_a == 0) d->bs_a = d->M * d->ld_a;
  if (d->bs_b == 0) d->bs_b = b_rows * d->ld_b;
  if (d->bs_d == 0) d->bs_d = d->N * d->ld_d;
  if (d->bs_e == 0) d->bs_e = d->M * d->ld_e;
  if (d->ld_a < d->K || d->ld_b < b_inner || d->ld_d < d->L || d->ld_e < d->L)
    return fail(MBCI_ERR_INVALID, "row stride smaller than the row");
  if (d->ld_a < 0 || d->ld_b < 0 || d->ld_d < 0 || d->ld_e < 0 || d->bs_a < 0 || d->bs_b < 0 ||
      d->bs_d < 0 || d->bs_e < 0)
    return fail(MBCI_ERR_INVALID, "negative stride");
  if (d->M > INT32_MAX || d->N > INT32_MAX || d->batch > INT32_MAX)
    return fail(MBCI_ERR_UNSUPPORTED, "dimension exceeds int32");
  if (std::isnan(d->scale))   // DESIGN.md R1 (scale, softmax) and R19 (activations: 1)
    d->scale = (d->op == MBCI_OP_RELU || d->op == MBCI_OP_GELU || d->K == 0) ? 1.0f
                                                                                : 1.0f / std::sqrt(static_cast<float>(d->K));
  return MBCI_OK;
}

int64_t span_elems(int64_t batch, int64_t rows, int64_t cols, int64_t ld, int64_t bs) {
  if (batch == 0 || rows == 0 || cols == 0) return 0;
  return (batch - 1) * bs + (rows - 1) * ld + cols;
}

// Kernel-5 feature flags (Tc4Params::flags); MBCI_T5_FLAGS overrides (diagnostics).
int t5_flags_default() {
  const char* e = getenv("MBCI_T5_FLAGS");
  if (e) return atoi(e) & 0x1FFF;
  return 7953;  // bit 0: exp-phase turns; bit 2: spinning single-thread waits (A/B only);
                // bits 4-5: hand the turn over that many 16-pair chunks before the end;
                // bit 8: event-driven issuers (G1 / G2 in whichever order their inputs arrive);
                // bit 9: linear ops convert S before waiting for P_x to be released
                // (C4 K = L = 16: 49.0 -> 44.4 us; softmax configs within noise, round 2);
                // bit 10: the epilogue sleeps between polls of its long O waits (~1 %);
                // bit 11: softmax warps poll s_full / p_free with test_wait on SOFTMAX (~1 %);
                // bit 12: P_x released first, each 16-column chunk of P stored as computed
                // (16 packed registers live instead of 64: C6 -2 %, C2 within noise)
}

// Kernel-4 feature flags (MBCI_T4_FLAGS overrides): bit 10 the epilogue sleeps between polls.
int t4_flags_default() {
  const char* e = getenv("MBCI_T4_FLAGS");
  if (e) return atoi(e) & 0x400;
  return 0;
}

// Kernel-6 feature flags (MBCI_T6_FLAGS overrides): bit 0 exp-phase turns between the slots,
// bit 4 hand the turn over one 16-pair chunk early, bit 2 spinning single-thread waits.
int t6_flags_default() {
  const char* e = getenv("MBCI_T6_FLAGS");
  if (e) return atoi(e) & 0x3F;
  return 1;
}

bool env_is(const char* name, const char* value) {
  const char* e = getenv(name);
  return e && strcmp(e, value) == 0;
}

// L2 prefetch budget per CTA of kernels 5 / 6 before the grid-dependency wait (MBCI_PF_KB
// overrides, 0 disables).
int pf_bytes_default() {
  const char* e = getenv("MBCI_PF_KB");
  if (e) return std::max(0, atoi(e)) * 1024;
  return 128 * 1024;
}

// Programmatic dependent launch for kernel 5 (MBCI_PDL=0 disables it, for A/B measurements).
bool pdl_enabled() {
  const char* e = getenv("MBCI_PDL");
  return !(e && e[0] == '0');
}

// Pairs of every 8 exponential pairs evaluated by the FMA-pipe polynomial in kernel 4
// (MBCI_T4_EMU overrides; 0 = all on the MUFU).
int t4_emu_default() {
  const char* e = getenv("MBCI_T4_EMU");
  if (e && (e[0] == '0' || e[0] == '2' || e[0] == '3' || e[0] == '4')) return e[0] - '0';
  return 2;   // 2/8 of the pairs: C2 21.0 us, C3 61.7 (3/8: 21.5, 63.1; 0: 22.2, 65.4; 4/8 slower)
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

mbci_status_t get_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) return fail(MBCI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return MBCI_OK;
}

// 3-D tiled map over [batch][rows][cols] (cols contiguous), box {64, box_rows, 1}, 128-B swizzle.
mbci_status_t encode3d(CUtensorMap* map, const void* base, bool bf16, int64_t cols, int64_t rows,
                       int64_t batch, int64_t ld, int64_t bs, uint32_t box_rows) {
  memset(map, 0, sizeof(*map));
  cuuint64_t dims[3] = {(cuuint64_t)std::max<int64_t>(cols, 1), (cuuint64_t)std::max<int64_t>(rows, 1),
                        (cuuint64_t)std::max<int64_t>(batch, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(std::max<int64_t>(ld, 8) * 2),
                           (cuuint64_t)(std::max<int64_t>(bs, 8) * 2)};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(MBCI_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): cols=%lld rows=%lld ld=%lld bs=%lld",
                (int)r, (long long)cols, (long long)rows, (long long)ld, (long long)bs);
  return MBCI_OK;
}

struct MapCacheEntry {
  const void *A = nullptr, *B = nullptr, *D = nullptr, *E = nullptr;
  CUtensorMap ta, tb, td, te;
  uint64_t stamp = 0;
};

}  // namespace

constexpr int kHostChunks = 8;   // run_host pipeline depth (batch chunks), at most

// run_host chunk count (MBCI_HOST_CHUNKS overrides, 1 = the serial single-stream pipeline)
int host_chunks() {
  const char* e = getenv("MBCI_HOST_CHUNKS");
  if (e) return std::max(1, std::min(kHostChunks, atoi(e)));
  return 4;
}

struct mbci_chain {
  mbci_chain_desc_t d{};
  mbci_plan_t plan{};
  int device = 0;
  // tensor-core path
  TcKernel tc = nullptr;
  TcParams tp{};
  Tc4Kernel tc4 = nullptr;   // kernel 4
  Tc5Kernel tc5 = nullptr;   // kernels 5 / 6 (same parameter block, plus E's tensor map)
  int32_t threads = 0;       // block size of the persistent kernels
  int32_t search_rounds = 0, search_measurements = 0;   // tune = 2 (Algorithm 1) statistics
  Tc4Params tp4{};
  Tf32Params tp7{};          // kernel 7 (fp32, 3xTF32)
  CUtensorMap tmF;           // chain3: F's tensor map (encoded per F pointer)
  const void* tmF_ptr = nullptr;
  bool chain3 = false;
  int32_t grid2 = 0;
  int32_t kch = 1, dch = 1;
  MapCacheEntry cache[16];   // tensor maps of the 16 most recent (A, B, D) pointer triples
  uint64_t stamp = 0;
  uint64_t* trace = nullptr;
  // end-to-end scratch
  void *dA = nullptr, *dB = nullptr, *dD = nullptr, *dE = nullptr;
  int32_t* dV = nullptr;
  size_t nA = 0, nB = 0, nD = 0, nE = 0;
  cudaStream_t cst[3] = {nullptr, nullptr, nullptr};   // run_host: H2D, kernels, D2H
  cudaEvent_t cev[3 + 2 * kHostChunks] = {};           // run_host: fork, per chunk (inputs in, kernel done), joins
  cudaGraphExec_t hg_exec = nullptr;                   // run_host: the captured chunk pipeline
  const void* hg_key[5] = {};                          // ... for these host pointers (A, B, D, E, valid_len)
  mbci_chain* sub[2] = {nullptr, nullptr};    // run_host: same plan on the chunk batch sizes
};

namespace {

int32_t elem_size(const mbci_chain_desc_t& d) { return d.dtype == MBCI_F32 ? 4 : 2; }

mbci_status_t setup_plan(mbci_chain* h) {
  const mbci_chain_desc_t& d = h->d;
  mbci_plan_t& p = h->plan;
  if (p.kernel == 0) {
    const int32_t k_steps = static_cast<int32_t>((d.K + 15) / 16);
    int32_t a_bytes, b_stage, d_stage;
    p.smem_bytes = static_cast<int32_t>(
        tc_smem_bytes(k_steps, p.BN, p.TL, p.stages, d.b_layout, &a_bytes, &b_stage, &d_stage));
    p.tmem_cols = tmem_alloc_cols(p.BN, p.TL);
    const bool stream = k_steps > 8;   // K > 128: live k loop (chain_tc.cuh, TcParams::kc)
    h->kch = stream ? 1 : std::max(1, (16 * k_steps + 63) / 64);
    h->dch = (p.TL + 63) / 64;
    h->tc = pick_tc(d.dtype == MBCI_BF16, p.BN, h->kch, d.b_layout, h->dch);
    TcParams& t = h->tp;
    t.M = (int32_t)d.M;
    t.N = (int32_t)d.N;
    t.K = (int32_t)d.K;
    t.L = (int32_t)d.L;
    t.batch = (int32_t)d.batch;
    t.l_m = (int32_t)((d.M + 127) / 128);
    t.l_h = (int32_t)((d.L + p.TL - 1) / p.TL);
    t.TL = p.TL;
    t.k_steps = k_steps;
    t.stages = p.stages;
    t.op = d.op;
    t.causal = (d.mask & MBCI_MASK_CAUSAL) ? 1 : 0;
    t.scale = d.op == MBCI_OP_SOFTMAX ? d.scale * 1.4426950408889634f : d.scale;
    t.ld_e = d.ld_e;
    t.bs_e = d.bs_e;
    t.a_bytes = (uint32_t)a_bytes;
    t.b_stage_bytes = (uint32_t)b_stage;
    t.d_stage_bytes = (uint32_t)d_stage;
    t.kp_rows = (uint32_t)(stream ? 64 : 16 * k_steps);
    t.kc = stream ? (int32_t)((d.K + 63) / 64) : 0;
    t.tmem_cols = (uint32_t)p.tmem_cols;
    const uint32_t fmt = d.dtype == MBCI_BF16 ? 1u : 0u;
    t.idesc1 = ptx::idesc_f16(fmt, 0, d.b_layout == 0 ? 1u : 0u, 128, (uint32_t)p.BN);
    t.idesc2 = ptx::idesc_f16(fmt, 0, 1u, 128, (uint32_t)p.TL);
    p.n_block = (int64_t)d.batch * t.l_m * t.l_h;
    if (p.n_block > INT32_MAX) return fail(MBCI_ERR_UNSUPPORTED, "kernel-0 grid exceeds 2^31 - 1 CTAs");
    cudaError_t e = cudaFuncSetAttribute((const void*)h->tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         p.smem_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  } else if (p.kernel == 4 || p.kernel == 5 || p.kernel == 6) {
    const int32_t k_steps = static_cast<int32_t>((d.K + 15) / 16);
    Tc4Layout lay;
    const bool fits = p.kernel >= 5 ? tc5_layout(k_steps, p.TL, p.stages, d.b_layout, &lay)
                                    : tc4_layout(k_steps, p.TL, p.stages, d.b_layout, &lay);
    if (k_steps < 1 || d.N < 1 || !fits)
      return fail(MBCI_ERR_UNSUPPORTED, "kernel-%d plan needs K, N >= 1 and must fit SMEM/TMEM", p.kernel);
    p.smem_bytes = lay.smem_total;
    p.tmem_cols = 512;
    h->kch = std::max(1, (16 * k_steps + 63) / 64);
    h->dch = (p.TL + 63) / 64;
    h->tc4 = nullptr;
    h->tc5 = nullptr;
    if (p.kernel == 5)
      // the linear ops run their own instantiation (EMU = -1), softmax the EMU variant
      h->tc5 = pick_tc5(d.dtype == MBCI_BF16, h->kch, d.b_layout,
                        d.op == MBCI_OP_SOFTMAX ? t4_emu_default() : -1);
    else if (p.kernel == 6)
      h->tc5 = pick_tc6(d.dtype == MBCI_BF16, h->kch, d.b_layout, t4_emu_default());
    else
      h->tc4 = pick_tc4(d.dtype == MBCI_BF16, h->kch, d.b_layout, h->dch, t4_emu_default());
    const void* kfn = p.kernel >= 5 ? (const void*)h->tc5 : (const void*)h->tc4;
    Tc4Params& t = h->tp4;
    t = Tc4Params{};
    t.M = (int32_t)d.M; t.N = (int32_t)d.N; t.K = (int32_t)d.K; t.L = (int32_t)d.L;
    t.batch = (int32_t)d.batch;
    t.l_mp = (int32_t)((d.M + 255) / 256);
    const int64_t units = (int64_t)d.batch * t.l_mp;
    if (units > INT32_MAX) return fail(MBCI_ERR_UNSUPPORTED, "kernel-4 unit count exceeds int32");
    t.units = (int32_t)units;
    t.TL = p.TL;
    t.k_steps = k_steps;
    t.stages = p.stages;
    t.q_bufs = lay.q_bufs;
    t.op = d.op;
    t.causal = (d.mask & MBCI_MASK_CAUSAL) ? 1 : 0;
    t.scale = d.op == MBCI_OP_SOFTMAX ? d.scale * 1.4426950408889634f : (d.op == MBCI_OP_NONE ? 1.0f : d.scale);
    t.ld_e = d.ld_e;
    t.bs_e = d.bs_e;
#if MBCI_TRACE
    // work-skipping diagnostics exist only in the trace build (libmbci_trace.so)
    if (const char* dbg = getenv("MBCI_T4_DEBUG")) t.dbg = atoi(dbg);
#endif
    t.q_bytes = (uint32_t)lay.q_bytes;
    t.b_stage_bytes = (uint32_t)lay.b_stage;
    t.d_stage_bytes = (uint32_t)lay.d_stage;
    t.kp_rows = (uint32_t)(16 * k_steps);
    const uint32_t fmt = d.dtype == MBCI_BF16 ? 1u : 0u;
    t.idesc1 = ptx::idesc_f16(fmt, 0, d.b_layout == 0 ? 1u : 0u, 128, 128u);
    t.idesc2 = ptx::idesc_f16(fmt, 0, 1u, 128, (uint32_t)p.TL);
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, h->device);
    // Wave quantisation: when the last, partial round has r <= n_sm / 2 units, each becomes two
    // "half" items (one 128-row Q tile, keys split between the two slots, merged in the CTA),
    // so the round takes half the tiles (chain_tc4.cuh).  Needs no key padding and an even
    // tile count; MBCI_T4_NO_HALF=1 disables it.
    t.nt_max = (int32_t)((d.N + 127) / 128);
    const int64_t rounds = units / n_sm, rem = units % n_sm;
    // (the two ring entries per step need stages >= 4 with three S buffers, >= 3 with two)
    const char* no_half = getenv("MBCI_T4_NO_HALF");
    const bool halves = rem > 0 && 2 * rem <= n_sm && t.nt_max % 2 == 0 && d.mask == MBCI_MASK_NONE &&
                        p.stages >= (h->dch == 1 ? 4 : 3) && !(no_half && no_half[0] == '1');
    t.half_from = halves ? (int32_t)(rounds * n_sm) : (int32_t)units;
    t.items = (int32_t)(halves ? t.half_from + 2 * rem : units);
    h->grid2 = (int32_t)std::max<int64_t>(1, std::min<int64_t>(n_sm, t.items));
    p.n_block = t.items;
    t.flags = p.kernel == 5 ? t5_flags_default() : (p.kernel == 6 ? t6_flags_default() : t4_flags_default());
    t.pf_bytes = p.kernel >= 5 ? pf_bytes_default() : 0;
    t.burst = (p.kernel >= 5 && !env_is("MBCI_T5_BURST", "0")) ? 1 : 0;
    h->threads = p.kernel == 6 ? kT6Threads : (p.kernel == 5 ? kT5Threads : kT4Threads);
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, h->threads,
                                                      p.smem_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
    if (occ < 1) return fail(MBCI_ERR_UNSUPPORTED, "kernel-%d CTA does not fit on an SM", p.kernel);
  } else if (p.kernel == 7) {
    if (d.dtype != MBCI_F32 || d.K < 1 || d.K > 128 || d.L > 128 || d.N < 1)
      return fail(MBCI_ERR_UNSUPPORTED, "kernel-7 plan needs fp32, 1 <= K <= 128, L <= 128, N >= 1");
    const bool wide = d.K > 64 || d.L > 64;   // 32-key tiles, 128 O columns (chain_tf32.cuh TfWide)
    Tf32Params& t = h->tp7;
    t = Tf32Params{};
    t.M = (int32_t)d.M; t.N = (int32_t)d.N; t.K = (int32_t)d.K; t.L = (int32_t)d.L;
    t.KP = (int32_t)((d.K + 7) / 8 * 8);
    t.TLP = (int32_t)std::max<int64_t>(16, (d.L + 15) / 16 * 16);
    t.op = d.op;
    t.causal = (d.mask & MBCI_MASK_CAUSAL) ? 1 : 0;
    t.scale = d.op == MBCI_OP_SOFTMAX ? d.scale * 1.4426950408889634f : (d.op == MBCI_OP_NONE ? 1.0f : d.scale);
    t.b_layout = d.b_layout;
    t.ld_a = d.ld_a; t.ld_b = d.ld_b; t.ld_d = d.ld_d; t.ld_e = d.ld_e;
    t.bs_a = d.bs_a; t.bs_b = d.bs_b; t.bs_d = d.bs_d; t.bs_e = d.bs_e;
    t.idesc1 = ptx::idesc_f16(2u, 0u, 0u, 128, wide ? 32u : 64u);   // kind::tf32: a/b format 2, K-major
    t.idesc2 = ptx::idesc_f16(2u, 0u, 0u, 128, (uint32_t)t.TLP);
    p.n_block = d.batch * ((d.M + 127) / 128);
    if (p.n_block > INT32_MAX) return fail(MBCI_ERR_UNSUPPORTED, "kernel-7 grid exceeds 2^31 - 1 CTAs");
    p.smem_bytes = (int32_t)(wide ? kTf32WideSmem : kTf32Smem);
    p.BN = wide ? 32 : 64;
    cudaError_t e = cudaFuncSetAttribute(tf32_fn(wide), cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  } else {
    if (d.batch * d.M > INT32_MAX) return fail(MBCI_ERR_UNSUPPORTED, "batch * M exceeds the CUDA-core grid");
    p.n_block = d.batch * d.M;
    const void* fn = simt_fn((int)d.dtype);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  }
  return MBCI_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

mbci_status_t launch(mbci_chain* h, const void* A, const void* B, const void* D, void* E,
                     const int32_t* valid_len, cudaStream_t st, float* lse = nullptr, int32_t key_off = 0) {
  const mbci_chain_desc_t& d = h->d;
  if (d.batch == 0 || d.M == 0 || d.L == 0) return MBCI_OK;  // nothing to write
  if (!E) return fail(MBCI_ERR_INVALID, "E is NULL");
  if (d.N > 0 && d.L > 0 && !D) return fail(MBCI_ERR_INVALID, "D is NULL");
  if (d.K > 0 && d.N > 0 && (!A || !B)) return fail(MBCI_ERR_INVALID, "A or B is NULL");
  if ((d.mask & MBCI_MASK_KEY_PADDING) && !valid_len)
    return fail(MBCI_ERR_INVALID, "mask KEY_PADDING needs valid_len");
  const int32_t* vl = (d.mask & MBCI_MASK_KEY_PADDING) ? valid_len : nullptr;
  if (h->plan.kernel == 0 || (h->plan.kernel >= 4 && h->plan.kernel <= 6)) {
    if (!aligned16(E) || (d.N > 0 && !aligned16(D)) || (d.K > 0 && d.N > 0 && (!aligned16(A) || !aligned16(B))))
      return fail(MBCI_ERR_UNSUPPORTED, "tensor-core path needs 16-byte aligned A, B, D, E");
    // tensor maps (cached by pointer triple)
    MapCacheEntry* ent = nullptr;
    for (auto& c : h->cache)
      if (c.stamp && c.A == A && c.B == B && c.D == D && c.E == E) ent = &c;
    if (!ent) {
      ent = &h->cache[0];
      for (auto& c : h->cache)
        if (c.stamp < ent->stamp) ent = &c;
      mbci_status_t s = get_encoder();
      if (s != MBCI_OK) return s;
      const bool bf16 = d.dtype == MBCI_BF16;
      memset(&ent->ta, 0, sizeof(CUtensorMap));
      memset(&ent->tb, 0, sizeof(CUtensorMap));
      memset(&ent->td, 0, sizeof(CUtensorMap));
      memset(&ent->te, 0, sizeof(CUtensorMap));
      const uint32_t bn_box = h->plan.kernel >= 4 ? 128u : (uint32_t)h->plan.BN;
      if (d.K > 0 && d.N > 0) {
        s = encode3d(&ent->ta, A, bf16, d.K, d.M, d.batch, d.ld_a, d.bs_a, 128);
        if (s != MBCI_OK) return s;
        const uint32_t kp_rows = h->plan.kernel == 0 ? h->tp.kp_rows : (uint32_t)(16 * ((d.K + 15) / 16));
        if (d.b_layout == 1)
          s = encode3d(&ent->tb, B, bf16, d.K, d.N, d.batch, d.ld_b, d.bs_b, bn_box);
        else
          s = encode3d(&ent->tb, B, bf16, d.N, d.K, d.batch, d.ld_b, d.bs_b, kp_rows);
        if (s != MBCI_OK) return s;
      }
      if (d.N > 0) {
        s = encode3d(&ent->td, D, bf16, d.L, d.N, d.batch, d.ld_d, d.bs_d, bn_box);
        if (s != MBCI_OK) return s;
      }
      if (h->plan.kernel >= 5) {   // E: TMA bulk stores of 128-row x 64-column tiles
        s = encode3d(&ent->te, E, bf16, d.L, d.M, d.batch, d.ld_e, d.bs_e, 128);
        if (s != MBCI_OK) return s;
      }
      ent->A = A;
      ent->B = B;
      ent->D = D;
      ent->E = E;
    }
    ent->stamp = ++h->stamp;
    if (h->plan.kernel == 0) {
      TcParams t = h->tp;
      t.valid_len = vl;
      t.key_off = key_off;
      t.lse = lse;
      t.E = E;
      t.trace = h->trace;
      h->tc<<<(unsigned)h->plan.n_block, kThreads, h->plan.smem_bytes, st>>>(ent->ta, ent->tb, ent->td,
                                                                          t.c3 ? h->tmF : ent->td, t);
    } else if (h->plan.kernel == 4) {
      Tc4Params t = h->tp4;
      t.valid_len = vl;
      t.key_off = key_off;
      t.lse = lse;
      t.E = E;
      t.trace = h->trace;
      h->tc4<<<(unsigned)h->grid2, kT4Threads, h->plan.smem_bytes, st>>>(ent->ta, ent->tb, ent->td, t);
    } else {
      Tc4Params t = h->tp4;
      t.valid_len = vl;
      t.key_off = key_off;
      t.lse = lse;
      t.E = E;
      t.trace = h->trace;
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3((unsigned)h->grid2);
      cfg.blockDim = dim3((unsigned)h->threads);
      cfg.dynamicSmemBytes = (size_t)h->plan.smem_bytes;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // chain_tc5.cuh header
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl_enabled() ? 1 : 0;
      cudaError_t le = cudaLaunchKernelEx(&cfg, h->tc5, ent->ta, ent->tb, ent->td, ent->te, t);
      if (le != cudaSuccess) return cuda_fail(le, "kernel-5/6 launch");
    }
  } else if (h->plan.kernel == 7) {
    Tf32Params t = h->tp7;
    t.valid_len = vl;
    t.key_off = key_off;
    t.lse = lse;
    cudaError_t le = launch_tf32(h->plan.BN == 32, (unsigned)h->plan.n_block, st, (const float*)A, (const float*)B,
                                 (const float*)D, (float*)E, t);
    if (le != cudaSuccess) return cuda_fail(le, "kernel-7 launch");
  } else {
    SimtParams sp{};
    sp.M = (int32_t)d.M;
    sp.N = (int32_t)d.N;
    sp.K = (int32_t)d.K;
    sp.L = (int32_t)d.L;
    sp.op = d.op;
    sp.causal = (d.mask & MBCI_MASK_CAUSAL) ? 1 : 0;
    sp.scale = d.scale;
    sp.b_layout = d.b_layout;
    sp.valid_len = vl;
    sp.key_off = key_off;
    sp.lse = lse;
    sp.ld_a = d.ld_a; sp.ld_b = d.ld_b; sp.ld_d = d.ld_d; sp.ld_e = d.ld_e;
    sp.bs_a = d.bs_a; sp.bs_b = d.bs_b; sp.bs_d = d.bs_d; sp.bs_e = d.bs_e;
    const unsigned grid = (unsigned)(d.batch * d.M);
    cudaError_t le = launch_simt((int)d.dtype, grid, h->plan.smem_bytes, st, A, B, D, E, sp);
    if (le != cudaSuccess) return cuda_fail(le, "CUDA-core kernel launch");
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return MBCI_OK;
}

mbci_status_t check_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= count) return fail(MBCI_ERR_INVALID, "device %d out of range (%d)", device, count);
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(MBCI_ERR_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major,
                prop.minor);
  return MBCI_OK;
}

// Seeded non-zero scratch inputs for tuning (equal scores would hide the rescale work):
// 16-bit normals via a counter hash + Box-Muller approximation-free mapping to [-2, 2).
__global__ void k_tune_fill(uint16_t* x, int64_t n, uint32_t seed, int bf16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    const float v = (float)((z >> 40) & 0xFFFFFF) * (4.0f / 16777216.0f) - 2.0f;
    x[i] = bf16 ? __bfloat16_as_ushort(__float2bfloat16(v)) : __half_as_ushort(__float2half(v));
  }
}

// Timing bench for plan selection (desc.tune = 1: measure a shortlist; 2: PAPER.md Alg. 1).
// Scratch inputs are seeded non-zero values; a candidate whose set-up or launch fails is never
// timed (+inf); a device fault poisons the context and is reported.
struct TuneBench {
  mbci_chain* h;
  void *A = nullptr, *B = nullptr, *D = nullptr, *E = nullptr;
  int32_t* V = nullptr;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  mbci_status_t fault = MBCI_OK;

  explicit TuneBench(mbci_chain* hh) : h(hh) {}
  mbci_status_t init() {
    const mbci_chain_desc_t& d = h->d;
    const int64_t s = elem_size(d);
    const int64_t b_rows = d.b_layout == 0 ? d.K : d.N, b_cols = d.b_layout == 0 ? d.N : d.K;
    const size_t nA = span_elems(d.batch, d.M, d.K, d.ld_a, d.bs_a) * s;
    const size_t nB = span_elems(d.batch, b_rows, b_cols, d.ld_b, d.bs_b) * s;
    const size_t nD = span_elems(d.batch, d.N, d.L, d.ld_d, d.bs_d) * s;
    const size_t nE = span_elems(d.batch, d.M, d.L, d.ld_e, d.bs_e) * s;
    if (cudaMalloc(&A, std::max<size_t>(nA, 16)) != cudaSuccess || cudaMalloc(&B, std::max<size_t>(nB, 16)) != cudaSuccess ||
        cudaMalloc(&D, std::max<size_t>(nD, 16)) != cudaSuccess || cudaMalloc(&E, std::max<size_t>(nE, 16)) != cudaSuccess ||
        cudaMalloc(&V, std::max<int64_t>(d.batch, 1) * 4) != cudaSuccess)
      return fail(MBCI_ERR_NOMEM, "tune scratch allocation failed");
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (s == 2) {
      k_tune_fill<<<256, 256, 0, st>>>((uint16_t*)A, (int64_t)(nA / 2), 1u, d.dtype == MBCI_BF16);
      k_tune_fill<<<256, 256, 0, st>>>((uint16_t*)B, (int64_t)(nB / 2), 2u, d.dtype == MBCI_BF16);
      k_tune_fill<<<256, 256, 0, st>>>((uint16_t*)D, (int64_t)(nD / 2), 3u, d.dtype == MBCI_BF16);
    } else {
      cudaMemsetAsync(A, 0, nA, st);
      cudaMemsetAsync(B, 0, nB, st);
      cudaMemsetAsync(D, 0, nD, st);
    }
    std::vector<int32_t> hv(std::max<int64_t>(d.batch, 1), (int32_t)d.N);
    cudaMemcpyAsync(V, hv.data(), hv.size() * 4, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    return MBCI_OK;
  }
  // seconds per launch of `plan` (2 warm-up + 5 timed launches), +inf if it cannot run
  double time_plan(const mbci_plan_t& plan) {
    if (fault != MBCI_OK) return 1e30;
    h->plan = plan;
    for (auto& c : h->cache) c = MapCacheEntry{};
    if (setup_plan(h) != MBCI_OK) return 1e30;
    bool ok = true;
    for (int w = 0; w < 2 && ok; ++w) ok = launch(h, A, B, D, E, V, st) == MBCI_OK;
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5 && ok; ++r) ok = launch(h, A, B, D, E, V, st) == MBCI_OK;
    cudaEventRecord(e1, st);
    cudaError_t ce = cudaEventSynchronize(e1);
    if (ce != cudaSuccess) {
      fault = cuda_fail(ce, "tuning run");
      return 1e30;
    }
    if (!ok || cudaGetLastError() != cudaSuccess) return 1e30;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e-3 / 5.0;
  }
  ~TuneBench() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (st) cudaStreamDestroy(st);
    cudaFree(A);
    cudaFree(B);
    cudaFree(D);
    cudaFree(E);
    cudaFree(V);
  }
};

mbci_status_t tune_plan(mbci_chain* h, const std::vector<mbci_plan_t>& plans) {
  // PAPER.md Alg. 1 lines 5-9 in one round: estimate all, measure the top n = 8.
  TuneBench tb(h);
  mbci_status_t rc = tb.init();
  if (rc != MBCI_OK) return rc;
  double best = 1e30;
  int best_i = -1;
  const int n_try = std::min<int>(8, (int)plans.size());
  for (int i = 0; i < n_try; ++i) {
    const double t = tb.time_plan(plans[i]);
    if (tb.fault != MBCI_OK) return tb.fault;
    if (t < best) {
      best = t;
      best_i = i;
    }
  }
  if (best_i < 0) return fail(MBCI_ERR_UNSUPPORTED, "tuning: no candidate plan launched successfully");
  h->plan = plans[best_i];
  for (auto& c : h->cache) c = MapCacheEntry{};
  return setup_plan(h);
}

// desc.tune = 2: PAPER.md Algorithm 1 over every legal plan, measured on the handle's device.
mbci_status_t search_plan(mbci_chain* h, const std::vector<mbci_plan_t>& plans) {
  TuneBench tb(h);
  mbci_status_t rc = tb.init();
  if (rc != MBCI_OK) return rc;
  SearchParams sp;   // N = 512, n = 8, eps = 1 %, seed 1, 64 rounds, the paper's t_estm
  mbci_plan_t best{};
  SearchLog log;
  const int r = alg1_search(plans, sp, [&](const mbci_plan_t& p) { return tb.time_plan(p); }, &best, &log);
  if (tb.fault != MBCI_OK) return tb.fault;
  if (r != 0 || log.best_measured >= 1e29) return fail(MBCI_ERR_UNSUPPORTED, "search: no candidate ran");
  h->plan = best;
  h->search_rounds = (int32_t)log.rounds.size();
  h->search_measurements = log.measurements;
  for (auto& c : h->cache) c = MapCacheEntry{};
  return setup_plan(h);
}

// Restores the caller's current device on scope exit (the ABI never leaves it changed).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

mbci_status_t create_impl(const mbci_chain_desc_t* desc, int device, const mbci_plan_t* forced,
                          mbci_chain_t* out) {
  if (!out) return fail(MBCI_ERR_INVALID, "out is NULL");
  *out = nullptr;
  mbci_chain_desc_t d;
  mbci_status_t s = normalize(desc, &d);
  if (s != MBCI_OK) return s;
  s = check_device(device);
  if (s != MBCI_OK) return s;
  DeviceGuard guard(device);
  mbci_hw_t hw;
  hw_default(&hw);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) {
    hw.n_sm = prop.multiProcessorCount;
    hw.smem_max = (int32_t)prop.sharedMemPerBlockOptin;
  }
  std::vector<mbci_plan_t> plans;
  enumerate_plans(d, hw, plans, /*rule3=*/forced == nullptr);
  if (plans.empty())
    return fail(MBCI_ERR_UNSUPPORTED, "no legal plan (N=%lld too large for the CUDA-core path?)", (long long)d.N);
  mbci_chain* h = new (std::nothrow) mbci_chain();
  if (!h) return fail(MBCI_ERR_NOMEM, "handle allocation failed");
  h->d = d;
  h->device = device;
  h->plan = plans[0];
  if (forced) {
    bool found = false;
    for (const auto& p : plans)
      if (p.kernel == forced->kernel && (p.kernel == 1 || p.kernel == 7 || (p.BN == forced->BN && p.TL == forced->TL &&
                                                           p.stages == forced->stages))) {
        h->plan = p;
        found = true;
      }
    if (!found) {
      delete h;
      return fail(MBCI_ERR_UNSUPPORTED, "forced plan (kernel=%d BN=%d TL=%d stages=%d) is not legal here",
                  forced->kernel, forced->BN, forced->TL, forced->stages);
    }
  }
  s = setup_plan(h);
  if (s == MBCI_OK && !forced && d.tune == 1 && plans.size() > 1) {
    // PAPER.md Alg. 1 lines 5-8: estimate every candidate, measure the top n = 8.
    // The shortlist keeps the best-ranked plans of every kernel family so that a model error
    // between families cannot hide the fastest kernel.
    std::vector<mbci_plan_t> shortlist;
    for (int fam : {7, 6, 5, 4, 0, 1}) {
      int taken = 0;
      for (const auto& q : plans)
        if (q.kernel == fam && taken < 3) {
          shortlist.push_back(q);
          ++taken;
        }
    }
    for (const auto& q : plans) {
      if ((int)shortlist.size() >= 8) break;
      bool dup = false;
      for (const auto& r : shortlist)
        dup |= (r.kernel == q.kernel && r.BN == q.BN && r.TL == q.TL && r.stages == q.stages);
      if (!dup) shortlist.push_back(q);
    }
    if (shortlist.size() > 8) shortlist.resize(8);
    s = tune_plan(h, shortlist);
  } else if (s == MBCI_OK && !forced && d.tune == 2 && plans.size() > 1) {
    s = search_plan(h, plans);   // PAPER.md Algorithm 1
  }
  if (s != MBCI_OK) {
    delete h;
    return s;
  }
  *out = h;
  return MBCI_OK;
}

}  // namespace

extern "C" {

mbci_status_t mbci_chain_create(const mbci_chain_desc_t* desc, int device, mbci_chain_t* out) {
  return create_impl(desc, device, nullptr, out);
}

mbci_status_t mbci_chain_create_with_plan(const mbci_chain_desc_t* desc, int device,
                                          const mbci_plan_t* plan, mbci_chain_t* out) {
  if (!plan) return fail(MBCI_ERR_INVALID, "plan is NULL");
  return create_impl(desc, device, plan, out);
}

mbci_status_t mbci_chain_run(mbci_chain_t h, const void* A, const void* B, const void* D, void* E,
                             const int32_t* valid_len, void* stream) {
  if (!h) return fail(MBCI_ERR_INVALID, "handle is NULL");
  DeviceGuard guard(h->device);   // launch on the handle's device, restore the caller's
  return launch(h, A, B, D, E, valid_len, reinterpret_cast<cudaStream_t>(stream));
}

mbci_status_t mbci_chain_run_partial(mbci_chain_t h, const void* A, const void* B, const void* D, void* E,
                                     float* lse, const int32_t* valid_len, int64_t key_offset, void* stream) {
  if (!h) return fail(MBCI_ERR_INVALID, "handle is NULL");
  if (key_offset < 0 || key_offset > INT32_MAX) return fail(MBCI_ERR_INVALID, "key_offset out of range");
  if (h->d.op == MBCI_OP_SOFTMAX && !lse && h->d.batch > 0 && h->d.M > 0)
    return fail(MBCI_ERR_INVALID, "SOFTMAX partial runs need lse");
  if (h->chain3) return fail(MBCI_ERR_UNSUPPORTED, "split-N partial runs of a three-contraction chain");
  if (h->d.mask & MBCI_MASK_CAUSAL) return fail(MBCI_ERR_UNSUPPORTED, "split-N partial runs with the causal mask");
  if (h->plan.kernel == 6) return fail(MBCI_ERR_UNSUPPORTED, "kernel 6 writes no log-sum-exp");
  DeviceGuard guard(h->device);
  return launch(h, A, B, D, E, valid_len, reinterpret_cast<cudaStream_t>(stream),
                h->d.op == MBCI_OP_SOFTMAX ? lse : nullptr, static_cast<int32_t>(key_offset));
}

mbci_status_t mbci_merge_partials(int32_t parts, const void* E_parts, const float* lse_parts, void* E, int64_t batch,
                                  int64_t M, int64_t L, int32_t dtype, int32_t op, void* stream) {
  if (parts < 1 || batch < 0 || M < 0 || L < 0 || dtype < 0 || dtype > 2 || op < 0 || op > 4)
    return fail(MBCI_ERR_INVALID, "bad merge arguments");
  if (batch == 0 || M == 0 || L == 0) return MBCI_OK;
  if (!E_parts || !E || (op == MBCI_OP_SOFTMAX && !lse_parts)) return fail(MBCI_ERR_INVALID, "NULL buffer");
  const int64_t rows = batch * M;
  const int64_t es = dtype == 0 ? 4 : 2, ve = 16 / es;
  const bool vec = L % ve == 0 && aligned16(E_parts) && aligned16(E);
  int dev = 0, n_sm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  const cudaError_t e = launch_merge(dtype, E_parts, lse_parts, E, parts, rows, L, op == MBCI_OP_SOFTMAX, vec, n_sm,
                                     reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "merge kernel launch");
  return MBCI_OK;
}

mbci_status_t mbci_chain_run_host(mbci_chain_t h, const void* A, const void* B, const void* D, void* E,
                                  const int32_t* valid_len, void* stream) {
  if (!h) return fail(MBCI_ERR_INVALID, "handle is NULL");
  const mbci_chain_desc_t& d = h->d;
  if (d.batch == 0 || d.M == 0 || d.L == 0) return MBCI_OK;
  if (!E) return fail(MBCI_ERR_INVALID, "E is NULL");
  if ((d.mask & MBCI_MASK_KEY_PADDING) && !valid_len) return fail(MBCI_ERR_INVALID, "mask KEY_PADDING needs valid_len");
  cudaStream_t ust = reinterpret_cast<cudaStream_t>(stream);
  const int64_t s = elem_size(d);
  const int64_t b_rows = d.b_layout == 0 ? d.K : d.N, b_cols = d.b_layout == 0 ? d.N : d.K;
  DeviceGuard guard(h->device);
  auto span_bytes = [&](int64_t nb, int64_t rows, int64_t cols, int64_t ld, int64_t bs) {
    return (size_t)(span_elems(nb, rows, cols, ld, bs) * s);
  };
  const size_t nA = span_bytes(d.batch, d.M, d.K, d.ld_a, d.bs_a), nB = span_bytes(d.batch, b_rows, b_cols, d.ld_b, d.bs_b);
  const size_t nD = span_bytes(d.batch, d.N, d.L, d.ld_d, d.bs_d), nE = span_bytes(d.batch, d.M, d.L, d.ld_e, d.bs_e);
  auto ensure = [&](void** p, size_t* have, size_t need) -> bool {
    if (*have >= need && *p) return true;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    if (cudaMalloc(p, std::max<size_t>(need, 16)) != cudaSuccess) return false;
    *have = need;
    return true;
  };
  size_t nV_have = h->dV ? (size_t)d.batch * 4 : 0;
  if (!ensure(&h->dA, &h->nA, nA) || !ensure(&h->dB, &h->nB, nB) || !ensure(&h->dD, &h->nD, nD) ||
      !ensure(&h->dE, &h->nE, nE) || !ensure((void**)&h->dV, &nV_have, (size_t)d.batch * 4))
    return fail(MBCI_ERR_NOMEM, "device scratch allocation failed");

  // Enqueue the copies and kernels of batch rows [b0, b0 + nb): H2D on s_in, the kernel on s_k
  // (after the inputs landed), D2H on s_out (after the kernel).  One stream for all three gives the
  // plain serial pipeline.
  auto enqueue = [&](mbci_chain* run, int64_t b0, int64_t nb, cudaStream_t s_in, cudaStream_t s_k,
                     cudaStream_t s_out, cudaEvent_t in_ev, cudaEvent_t k_ev) -> mbci_status_t {
    cudaError_t e = cudaSuccess;
    auto h2d = [&](void* dst, const void* src, int64_t rows, int64_t cols, int64_t ld, int64_t bs) {
      const size_t off = (size_t)(b0 * bs * s), len = span_bytes(nb, rows, cols, ld, bs);
      if (len && e == cudaSuccess)
        e = cudaMemcpyAsync((char*)dst + off, (const char*)src + off, len, cudaMemcpyHostToDevice, s_in);
    };
    if (d.K > 0 && d.N > 0) {
      h2d(h->dA, A, d.M, d.K, d.ld_a, d.bs_a);
      h2d(h->dB, B, b_rows, b_cols, d.ld_b, d.bs_b);
    }
    if (d.N > 0) h2d(h->dD, D, d.N, d.L, d.ld_d, d.bs_d);
    const int32_t* dv = nullptr;
    if (d.mask & MBCI_MASK_KEY_PADDING) {
      if (e == cudaSuccess) e = cudaMemcpyAsync(h->dV + b0, valid_len + b0, nb * 4, cudaMemcpyHostToDevice, s_in);
      dv = h->dV + b0;
    }
    if (e != cudaSuccess) return cuda_fail(e, "run_host H2D");
    if (s_k != s_in) {
      cudaEventRecord(in_ev, s_in);
      cudaStreamWaitEvent(s_k, in_ev, 0);
    }
    mbci_status_t rs = launch(run, (const char*)h->dA + b0 * d.bs_a * s, (const char*)h->dB + b0 * d.bs_b * s,
                              (const char*)h->dD + b0 * d.bs_d * s, (char*)h->dE + b0 * d.bs_e * s, dv, s_k);
    if (rs != MBCI_OK) return rs;
    if (s_out != s_k) {
      cudaEventRecord(k_ev, s_k);
      cudaStreamWaitEvent(s_out, k_ev, 0);
    }
    // E back row by row (2-D copies) so host bytes between rows are never written
    char* he = (char*)E + b0 * d.bs_e * s;
    const char* de = (const char*)h->dE + b0 * d.bs_e * s;
    if (d.bs_e == d.M * d.ld_e) {
      e = cudaMemcpy2DAsync(he, d.ld_e * s, de, d.ld_e * s, d.L * s, nb * d.M, cudaMemcpyDeviceToHost, s_out);
    } else {
      for (int64_t b = 0; b < nb && e == cudaSuccess; ++b)
        e = cudaMemcpy2DAsync(he + b * d.bs_e * s, d.ld_e * s, de + b * d.bs_e * s, d.ld_e * s, d.L * s, d.M,
                              cudaMemcpyDeviceToHost, s_out);
    }
    if (e != cudaSuccess) return cuda_fail(e, "run_host D2H E");
    return MBCI_OK;
  };

  // Pinned host buffers: the batch is cut into up to kHostChunks chunks pipelined over three
  // handle-owned streams (all H2D copies back to back — PCIe-bound —, each chunk's kernel once its
  // inputs landed, each chunk's D2H once its kernel ran), captured ONCE into a CUDA graph per set of
  // host pointers and replayed on `stream`: one graph launch per call instead of ~8 API calls per
  // chunk.  A chunk runs the handle's plan on its batch rows through a sub-handle (created once).
  auto pinned = [](const void* p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool graph_ok = pinned(A) && pinned(B) && pinned(D) && pinned(E) &&
                        (!(d.mask & MBCI_MASK_KEY_PADDING) || pinned(valid_len)) && host_chunks() > 1;
  if (graph_ok) {
    const void* key[5] = {A, B, D, E, valid_len};
    bool hit = h->hg_exec != nullptr;
    for (int i = 0; i < 5 && hit; ++i) hit = h->hg_key[i] == key[i];
    if (!hit) {
      if (h->hg_exec) {
        cudaGraphExecDestroy(h->hg_exec);
        h->hg_exec = nullptr;
      }
      const int64_t n_chunks = std::min<int64_t>(d.batch, host_chunks());
      const int64_t cb = (d.batch + n_chunks - 1) / n_chunks;
      for (int i = 0; i < 3; ++i)
        if (!h->cst[i] && cudaStreamCreateWithFlags(&h->cst[i], cudaStreamNonBlocking) != cudaSuccess)
          return fail(MBCI_ERR_CUDA, "stream creation failed");
      for (auto& ev : h->cev)
        if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
          return fail(MBCI_ERR_CUDA, "event creation failed");
      // sub-handles first (host work, outside the capture)
      std::vector<mbci_chain*> runs;
      for (int64_t c = 0; c < n_chunks; ++c) {
        const int64_t nb = std::min(cb, d.batch - c * cb);
        if (nb <= 0) break;
        mbci_chain* sub = nullptr;
        for (auto& sh : h->sub)
          if (sh && sh->d.batch == nb) sub = sh;
        if (!sub) {
          mbci_chain_desc_t sd = d;
          sd.batch = nb;
          sd.tune = 0;
          mbci_chain_t nh = nullptr;
          mbci_status_t rs = create_impl(&sd, h->device, &h->plan, &nh);
          if (rs != MBCI_OK) return rs;
          for (auto& sh : h->sub)
            if (!sh) { sh = nh; nh = nullptr; break; }
          if (nh) {
            mbci_chain_destroy(nh);
            return fail(MBCI_ERR_CUDA, "run_host: sub-handle cache full");
          }
          sub = h->sub[0]->d.batch == nb ? h->sub[0] : h->sub[1];
        }
        runs.push_back(sub);
      }
      cudaError_t ce = cudaStreamBeginCapture(h->cst[0], cudaStreamCaptureModeThreadLocal);
      if (ce != cudaSuccess) return cuda_fail(ce, "run_host graph capture");
      cudaEventRecord(h->cev[0], h->cst[0]);
      cudaStreamWaitEvent(h->cst[1], h->cev[0], 0);
      cudaStreamWaitEvent(h->cst[2], h->cev[0], 0);
      mbci_status_t rs = MBCI_OK;
      for (size_t c = 0; c < runs.size() && rs == MBCI_OK; ++c)
        rs = enqueue(runs[c], (int64_t)c * cb, runs[c]->d.batch, h->cst[0], h->cst[1], h->cst[2], h->cev[1 + 2 * c],
                     h->cev[2 + 2 * c]);
      // rejoin the forked streams into the capture origin
      cudaEventRecord(h->cev[2 * kHostChunks + 1], h->cst[1]);
      cudaEventRecord(h->cev[2 * kHostChunks + 2], h->cst[2]);
      cudaStreamWaitEvent(h->cst[0], h->cev[2 * kHostChunks + 1], 0);
      cudaStreamWaitEvent(h->cst[0], h->cev[2 * kHostChunks + 2], 0);
      cudaGraph_t g = nullptr;
      ce = cudaStreamEndCapture(h->cst[0], &g);
      if (rs != MBCI_OK) {
        if (g) cudaGraphDestroy(g);
        return rs;
      }
      if (ce != cudaSuccess || !g) return cuda_fail(ce, "run_host graph capture");
      ce = cudaGraphInstantiate(&h->hg_exec, g, 0);
      cudaGraphDestroy(g);
      if (ce != cudaSuccess) {
        h->hg_exec = nullptr;
        return cuda_fail(ce, "run_host graph instantiate");
      }
      for (int i = 0; i < 5; ++i) h->hg_key[i] = key[i];
    }
    cudaError_t e = cudaGraphLaunch(h->hg_exec, ust);
    if (e != cudaSuccess) return cuda_fail(e, "run_host graph launch");
    e = cudaStreamSynchronize(ust);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    return MBCI_OK;
  }
  // pageable host memory: the serial pipeline on `stream`
  mbci_status_t rs = enqueue(h, 0, d.batch, ust, ust, ust, nullptr, nullptr);
  if (rs != MBCI_OK) return rs;
  cudaError_t e = cudaStreamSynchronize(ust);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  return MBCI_OK;
}

// ---- three-contraction chains (R20) --------------------------------
mbci_status_t mbci_chain3_create(const mbci_chain3_desc_t* desc3, int device, mbci_chain_t* out) {
  if (!desc3 || !out) return fail(MBCI_ERR_INVALID, "NULL argument");
  *out = nullptr;
  const mbci_chain3_desc_t& c = *desc3;
  if (c.H < 0) return fail(MBCI_ERR_INVALID, "negative H");
  if (c.op2 != MBCI_OP_NONE && c.op2 != MBCI_OP_SCALE && c.op2 != MBCI_OP_RELU && c.op2 != MBCI_OP_GELU)
    return fail(MBCI_ERR_INVALID, "op2 must be NONE, SCALE, RELU or GELU");
  mbci_chain_desc_t d{};
  d.batch = c.batch; d.M = c.M; d.N = c.N; d.K = c.K; d.L = c.L;
  d.dtype = c.dtype; d.op = c.op; d.scale = c.scale; d.mask = c.mask; d.b_layout = c.b_layout;
  d.ld_e = c.H;
  d.bs_e = c.M * c.H;
  mbci_chain_desc_t n;
  mbci_status_t s = normalize(&d, &n);
  if (s != MBCI_OK) return s;
  if (n.dtype == MBCI_F32) return fail(MBCI_ERR_UNSUPPORTED, "chain3 takes fp16 / bf16");
  if (n.L < 1 || n.L > 128) return fail(MBCI_ERR_UNSUPPORTED, "chain3 keeps the intermediate on chip: 1 <= L <= 128");
  if (!tc_eligible(n) || c.H % 8 != 0) return fail(MBCI_ERR_UNSUPPORTED, "chain3 needs 16-byte rows (K, N, L, H % 8)");
  s = check_device(device);
  if (s != MBCI_OK) return s;
  DeviceGuard guard(device);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return fail(MBCI_ERR_CUDA, "device properties");
  const int32_t k_steps = static_cast<int32_t>((n.K + 15) / 16);
  const int32_t lpad = static_cast<int32_t>(std::max<int64_t>(16, (n.L + 15) / 16 * 16));
  // plan: kernel 0, the whole L per CTA (TL = L padded), H in TH-column chunks on the grid
  mbci_plan_t best{};
  bool found = false;
  for (int32_t BN : {128, 64}) {
    for (int32_t TH : {128, 64}) {
      if (TH > 64 && c.H <= 64) continue;
      const int32_t cols = 2 * BN + lpad + TH;
      if (cols > 512) continue;
      for (int32_t st = 4; st >= 2 && !found; --st) {
        const int64_t f_bytes = (int64_t)(TH / 64) * lpad * 128;
        const int64_t smem = tc_smem_bytes(k_steps, BN, lpad, st, n.b_layout, nullptr, nullptr, nullptr) + 1024 + f_bytes;
        if (smem > prop.sharedMemPerBlockOptin) continue;
        best = mbci_plan_t{};
        best.kernel = 0; best.BM = 128; best.BN = BN; best.TK = 16 * std::max(1, k_steps); best.TL = lpad;
        best.stages = st; best.smem_bytes = (int32_t)smem; best.tmem_cols = cols;
        found = true;
      }
      if (found) {
        mbci_chain* h = new (std::nothrow) mbci_chain();
        if (!h) return fail(MBCI_ERR_NOMEM, "handle allocation failed");
        h->d = n;
        h->device = device;
        h->plan = best;
        h->chain3 = true;
        s = setup_plan(h);
        if (s != MBCI_OK) {
          delete h;
          return s;
        }
        TcParams& t = h->tp;
        t.c3 = 1;
        t.H = (int32_t)c.H;
        t.TH = TH;
        t.op2 = c.op2;
        t.scale2 = c.op2 == MBCI_OP_NONE ? 1.0f : (std::isnan(c.scale2) ? 1.0f : c.scale2);
        t.f_bytes = (uint32_t)((TH / 64) * lpad * 128);
        t.idesc3 = ptx::idesc_f16(n.dtype == MBCI_BF16 ? 1u : 0u, 0, 1u, 128, (uint32_t)TH);
        t.l_h = (int32_t)((c.H + TH - 1) / TH);
        int32_t tc = 32;
        while (tc < 2 * BN + lpad + TH) tc <<= 1;
        t.tmem_cols = (uint32_t)tc;
        h->plan.tmem_cols = tc;
        h->plan.smem_bytes = best.smem_bytes;
        h->plan.n_block = n.batch * t.l_m * t.l_h;
        if (h->plan.n_block > INT32_MAX) {
          delete h;
          return fail(MBCI_ERR_UNSUPPORTED, "chain3 grid exceeds 2^31 - 1 CTAs");
        }
        cudaError_t e = cudaFuncSetAttribute((const void*)h->tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             h->plan.smem_bytes);
        if (e != cudaSuccess) {
          delete h;
          return cuda_fail(e, "cudaFuncSetAttribute");
        }
        *out = h;
        return MBCI_OK;
      }
    }
  }
  return fail(MBCI_ERR_UNSUPPORTED, "chain3: no plan fits shared / tensor memory");
}

mbci_status_t mbci_chain3_run(mbci_chain_t h, const void* A, const void* B, const void* D, const void* F, void* E,
                              const int32_t* valid_len, void* stream) {
  if (!h || !h->chain3) return fail(MBCI_ERR_INVALID, "not a chain3 handle");
  const mbci_chain_desc_t& d = h->d;
  if (d.batch == 0 || d.M == 0 || h->tp.H == 0) return MBCI_OK;
  if (d.N > 0 && !F) return fail(MBCI_ERR_INVALID, "F is NULL");
  if (F && !aligned16(F)) return fail(MBCI_ERR_UNSUPPORTED, "F must be 16-byte aligned");
  DeviceGuard guard(h->device);
  if (d.N > 0 && F != h->tmF_ptr) {
    mbci_status_t s = get_encoder();
    if (s != MBCI_OK) return s;
    s = encode3d(&h->tmF, F, d.dtype == MBCI_BF16, h->tp.H, d.L, d.batch, h->tp.H, d.L * h->tp.H,
                 (uint32_t)h->tp.TL);
    if (s != MBCI_OK) return s;
    h->tmF_ptr = F;
  }
  return launch(h, A, B, D, E, valid_len, reinterpret_cast<cudaStream_t>(stream));
}

mbci_status_t mbci_chain_destroy(mbci_chain_t h) {
  if (!h) return MBCI_OK;
  for (auto& sh : h->sub) mbci_chain_destroy(sh);
  for (auto& c : h->cst)
    if (c) cudaStreamDestroy(c);
  for (auto& ev : h->cev)
    if (ev) cudaEventDestroy(ev);
  if (h->hg_exec) cudaGraphExecDestroy(h->hg_exec);
  cudaFree(h->dA);
  cudaFree(h->dB);
  cudaFree(h->dD);
  cudaFree(h->dE);
  cudaFree(h->dV);
  delete h;
  return MBCI_OK;
}

mbci_status_t mbci_chain_plan(mbci_chain_t h, mbci_plan_t* out) {
  if (!h || !out) return fail(MBCI_ERR_INVALID, "NULL argument");
  *out = h->plan;
  return MBCI_OK;
}

mbci_status_t mbci_chain_describe(mbci_chain_t h, char* buf, size_t len) {
  if (!h || !buf || len == 0) return fail(MBCI_ERR_INVALID, "NULL argument");
  const mbci_plan_t& p = h->plan;
  snprintf(buf, len,
           "kernel=%s BM=%d BN=%d TK=%d TL=%d stages=%d smem=%d tmem=%d n_block=%lld "
           "t_estm=%.3gs alpha=%.4f t_b200=%.3gs",
           p.kernel == 0 ? "tcgen05" : (p.kernel == 4 ? "tcgen05-pingpong" : (p.kernel == 5 ? "tcgen05-pingpong-sepP" : (p.kernel == 6 ? "tcgen05-pingpong-splitrow" : (p.kernel == 7 ? "tcgen05-tf32x3" : "simt")))), p.BM, p.BN, p.TK, p.TL, p.stages, p.smem_bytes, p.tmem_cols,
           (long long)p.n_block, p.t_estm, p.alpha, p.t_b200);
  return MBCI_OK;
}

mbci_status_t mbci_chain_set_trace(mbci_chain_t h, void* buf, int64_t cap_bytes) {
  if (!h) return fail(MBCI_ERR_INVALID, "handle is NULL");
  const int64_t need = (h->plan.kernel >= 4 && h->plan.kernel <= 6) ? (int64_t)h->grid2 * kT4TraceSlots * 8
                                             : h->plan.n_block * kTraceSlots * 8;
  if (buf && cap_bytes < need) return fail(MBCI_ERR_INVALID, "trace buffer needs %lld bytes", (long long)need);
  h->trace = static_cast<uint64_t*>(buf);
  return MBCI_OK;
}

int32_t mbci_chain_launches_per_run(mbci_chain_t h) {
  if (!h) return 0;
  return (h->d.batch == 0 || h->d.M == 0 || h->d.L == 0) ? 0 : 1;
}

const char* mbci_status_string(mbci_status_t s) {
  switch (s) {
    case MBCI_OK: return "MBCI_OK";
    case MBCI_ERR_INVALID: return "MBCI_ERR_INVALID";
    case MBCI_ERR_UNSUPPORTED: return "MBCI_ERR_UNSUPPORTED";
    case MBCI_ERR_CUDA: return "MBCI_ERR_CUDA";
    case MBCI_ERR_NOMEM: return "MBCI_ERR_NOMEM";
  }
  return "MBCI_ERR_?";
}

const char* mbci_last_error(void) { return g_err.c_str(); }

int32_t mbci_abi_version(void) { return MBCI_ABI_VERSION; }

void mbci_hw_default(mbci_hw_t* hw) {
  if (hw) hw_default(hw);
}

mbci_status_t mbci_plan_enumerate(const mbci_chain_desc_t* desc, const mbci_hw_t* hw, mbci_plan_t* plans,
                                  int32_t cap, int32_t* n_out) {
  mbci_chain_desc_t d;
  mbci_status_t s = normalize(desc, &d);
  if (s != MBCI_OK) return s;
  mbci_hw_t h;
  if (hw) h = *hw; else hw_default(&h);
  std::vector<mbci_plan_t> v;
  enumerate_plans(d, h, v);
  if (n_out) *n_out = (int32_t)v.size();
  if (plans)
    for (int32_t i = 0; i < cap && i < (int32_t)v.size(); ++i) plans[i] = v[i];
  if (v.empty()) return fail(MBCI_ERR_UNSUPPORTED, "no legal plan");
  return MBCI_OK;
}

mbci_status_t mbci_plan_select(const mbci_chain_desc_t* desc, const mbci_hw_t* hw, mbci_plan_t* out) {
  if (!out) return fail(MBCI_ERR_INVALID, "out is NULL");
  int32_t n = 0;
  return mbci_plan_enumerate(desc, hw, out, 1, &n);
}

mbci_status_t mbci_plan_search(const mbci_chain_desc_t* desc, const mbci_hw_t* hw,
                               const mbci_search_params_t* params, mbci_measure_fn measure, void* user,
                               mbci_plan_t* best, mbci_search_result_t* result, double* round_log) {
  if (!measure || !best) return fail(MBCI_ERR_INVALID, "measure and best must be non-NULL");
  mbci_chain_desc_t d;
  mbci_status_t s = normalize(desc, &d);
  if (s != MBCI_OK) return s;
  mbci_hw_t hh;
  if (hw) hh = *hw; else hw_default(&hh);
  std::vector<mbci_plan_t> space;
  enumerate_plans(d, hh, space);
  if (space.empty()) return fail(MBCI_ERR_UNSUPPORTED, "no legal plan");
  SearchParams sp;
  if (params) {
    sp.N = params->N;
    sp.n = params->n;
    sp.eps = params->eps;
    sp.seed = params->seed;
    sp.max_rounds = params->max_rounds;
    sp.model = params->model;
  }
  SearchLog log;
  const int r = alg1_search(space, sp, [&](const mbci_plan_t& p) { return measure(&p, user); }, best, &log);
  if (r != 0) return fail(MBCI_ERR_INVALID, "bad search parameters");
  if (result) {
    result->rounds = (int32_t)log.rounds.size();
    result->measurements = log.measurements;
    result->space_size = (int32_t)space.size();
    result->best_measured = log.best_measured;
    result->history_min = log.history_min;
  }
  if (round_log)
    for (size_t i = 0; i < log.rounds.size(); ++i) {
      round_log[3 * i] = log.rounds[i].best_estimated;
      round_log[3 * i + 1] = log.rounds[i].top1_measured;
      round_log[3 * i + 2] = log.rounds[i].best_measured;
    }
  return MBCI_OK;
}

mbci_status_t mbci_chain_search_stats(mbci_chain_t h, int32_t* rounds, int32_t* measurements) {
  if (!h) return fail(MBCI_ERR_INVALID, "handle is NULL");
  if (rounds) *rounds = h->search_rounds;
  if (measurements) *measurements = h->search_measurements;
  return MBCI_OK;
}

mbci_status_t mbci_model_terms(int64_t batch, int64_t M, int64_t N, int64_t K, int64_t L, int64_t TM,
                               int64_t TN, int64_t TK, int64_t TH, int32_t elem_bytes, const mbci_hw_t* hw,
                               double out[5]) {
  if (!out || TM <= 0 || TN <= 0 || TK <= 0 || TH <= 0 || batch <= 0 || M < 0 || N < 0 || K < 0 || L < 0 ||
      elem_bytes <= 0)
    return fail(MBCI_ERR_INVALID, "bad model arguments");
  mbci_hw_t h;
  if (hw) h = *hw; else hw_default(&h);
  model_terms(batch, M, N, K, L, TM, TN, TK, TH, elem_bytes, h, out);
  return MBCI_OK;
}

mbci_status_t mbci_prune_funnel(int64_t M, int64_t N, int64_t K, int64_t H, int32_t elem_bytes, int64_t shm_max,
                                mbci_funnel_t* out) {
  if (!out || M <= 0 || N <= 0 || K <= 0 || H <= 0 || elem_bytes <= 0 || shm_max <= 0)
    return fail(MBCI_ERR_INVALID, "bad funnel arguments");
  const mbci_status_t st = prune_funnel(M, N, K, H, elem_bytes, shm_max, out);
  if (st != MBCI_OK) return fail(st, "more than 2^30 tile vectors survive Rule 3");
  return MBCI_OK;
}

}  // extern "C"
