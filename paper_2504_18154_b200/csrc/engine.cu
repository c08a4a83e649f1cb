// The PaDG instance engine behind include/ecoserve.h: KV block allocator and
// block tables, weight preparation, and the two phase
// executors that temporal disaggregation alternates between (PAPER.md Sec.
// 3.2.1):
//   prefill phase  (a6-a12): embed -> L x [RMSNorm, QKV GEMM + RoPE + KV write,
//                  causal varlen attention, O GEMM + residual, RMSNorm,
//                  gate/up GEMM + SiLU*up, down GEMM + residual] -> final norm of
//                  each sequence's last row -> LM head + greedy argmax
//   decode phase   (a13-a16): the same per step with B rows, skinny split-K
//                  "swap-AB" GEMMs (weights on the MMA M side), split-K paged
//                  attention, continuous batching (finished requests leave).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <unordered_map>
#include <chrono>
#include <vector>

#include <nccl.h>

#include "../../include/ecoserve.h"
#include "kernels.h"

using namespace eco;

namespace {

constexpr int BLOCK = 64;
constexpr int BN_PREFILL = 256;

struct Req {
  int64_t id;
  std::vector<int> prompt;
  int S = 0;
  int max_new = 1;
  int n_gen = 0;
  int last_token = -1;
  bool finished = false;
  int prefilled = 0;  // prompt tokens whose K / V are in the pool (chunked prefill)
  std::vector<int> blocks;
};

struct ActMaps {  // one activation buffer as GEMM operand
  CUtensorMap a;          // as A (box 128 rows): prefill
  CUtensorMap b[3];       // as B with box 64 / 128 / 256 rows: decode (swap-AB)
};

struct LayerW {
  const bf16 *attn_norm, *ffn_norm, *wo, *wd;
  bf16 *wqkv, *wgu;
  CUtensorMap qkv_a, qkv_b, o_a, o_b, gu_a, gu_b, d_a, d_b;  // _a: box 128 (decode A), _b: box 256 (prefill B)
  // decode gate/up in two waves (gu2_a: the tiles past the first wave) and the down
  // projection split at that K boundary (d1_a: K blocks [0, W1), d2_a: [W1, F/64))
  CUtensorMap gu2_a, d1_a, d2_a;
};

int bn_index(int bn) { return bn == 64 ? 0 : bn == 128 ? 1 : 2; }
int pick_bn(int rows) { return rows <= 64 ? 64 : rows <= 128 ? 128 : 256; }

// CUDA-event profiler on the instance stream (ecoserve_get_timing).
enum ProfClass { P_PREFILL = 0, P_DECODE, P_GEMM_PREFILL, P_GEMM_DECODE, P_ATTN_PREFILL, P_ATTN_DECODE, P_OTHER, P_N };

struct Prof {
  int level = 1;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Mark {
    cudaEvent_t a, b;
    int cls;
    double work;
  };
  std::vector<Mark> marks;
  double ms[P_N] = {0}, work[P_N] = {0};
  int64_t count[P_N] = {0};
  int64_t tokens[2] = {0, 0};
  int64_t launches = 0;
  int64_t h2d = 0, d2h = 0;

  cudaEvent_t get() {
    if (used == pool.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      pool.push_back(e);
    }
    return pool[used++];
  }
  // returns the mark index or -1
  int begin(int cls, cudaStream_t s) {
    if (level == 0 || (cls >= P_GEMM_PREFILL && level < 2)) return -1;
    Mark m{get(), get(), cls, 0.0};
    if (!m.a || !m.b) return -1;
    cudaEventRecord(m.a, s);
    marks.push_back(m);
    return (int)marks.size() - 1;
  }
  void end(int idx, double w, cudaStream_t s) {
    if (idx < 0) return;
    marks[idx].work = w;
    cudaEventRecord(marks[idx].b, s);
  }
  // after a stream sync
  void resolve() {
    for (auto& m : marks) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, m.a, m.b) == cudaSuccess) {
        ms[m.cls] += t;
        work[m.cls] += m.work;
        count[m.cls] += 1;
      }
    }
    marks.clear();
    used = 0;
  }
  void reset() {
    for (int i = 0; i < P_N; ++i) ms[i] = work[i] = 0, count[i] = 0;
    tokens[0] = tokens[1] = 0;
    launches = 0;
    h2d = d2h = 0;
  }
};

}  // namespace

struct ecoserve_instance {
  ecoserve_model_shape shape{};
  int L = 0, H = 0, M = 0, Mkv = 0, D = 0, F = 0, V = 0, QKV = 0;
  int device = 0, num_sms = 148;
  int tp = 1, tp_rank = 0;
  ncclComm_t comm = nullptr;     // TP=2 pair (a17): all-reduce of the residual after O and down
  // fused TP all-reduce over NVLink peer memory (N2): receive rows / flags written by the peer
  bool tp_fused = false;
  int tp_rows_max = 0, tp_epoch = 0;
  int* tp_err = nullptr;         // device flag: a TP exchange wait timed out (peer gone)
  int* h_tp_err = nullptr;       // pinned copy, read after every step
  unsigned long long tp_timeout_ns = 0;
  float* tp_recv = nullptr;      // [2 parity][2 rank][tp_rows_max][H]: both ranks' O / down outputs
  int* tp_flags = nullptr;       // [0]: epoch of the peer's last GEMM push; [64 + par * rows_max + row]: decode row flags
  float* peer_recv = nullptr;    // the peer's tp_recv / tp_flags (peer pointer or IPC mapping)
  int* peer_flags = nullptr;
  bool peer_ipc = false;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool dead = false;
  std::string err;
  // config
  int T_max = 16384, B_max = 512, P_max = 16384;
  bool debug = false;
  // pool
  bf16* pool = nullptr;
  int64_t num_blocks = 0;
  int64_t blk_stride = 0;  // elements per physical block (all layers)
  std::vector<int> free_blocks;
  // weights
  const bf16 *embed = nullptr, *lm_head = nullptr, *final_norm = nullptr;
  std::vector<LayerW> lw;
  CUtensorMap lm_a;
  CUtensorMap* d_wmaps = nullptr;  // device copies: [L][4] (qkv_a, o_a, gu_a, d_a) then lm_a (L2 prefetch)
  bool attn_tc = false;          // tcgen05 prefill attention (head_dim 128) in use
  CUtensorMap attn_qmap, attn_kvmap;
  // workspace
  float* x = nullptr;            // [T_max][H] residual stream
  bf16* h = nullptr;             // [T_max][H] normed GEMM input
  bf16* q = nullptr;             // [T_max][M][D]
  bf16* ao = nullptr;            // [T_max][M*D] attention output
  bf16* act = nullptr;           // [T_max][F]
  bf16* hl = nullptr;            // [B_max][H] final-normed last rows
  ActMaps m_h, m_ao, m_act, m_hl;
  float* part = nullptr;         // split-K partials
  int64_t part_elems = 0;
  int* counters = nullptr;       // split-K tile arrival counters
  float* attn_ws = nullptr;      // decode attention partials
  int64_t attn_ws_elems = 0;
  float* am_val = nullptr;
  int* am_idx = nullptr;
  int am_ld = 0;
  int* d_tokens = nullptr;
  int* sk_cnt = nullptr;         // [B_max * Mkv] stream-K decode attention item counters (zero at rest)
  float* nrm_ss = nullptr;       // [ceil(H/256)][T_max] prefill deferred RMSNorm: per-tile sums of x^2
  // decode gate/up second wave beside the down projection's first K part (gu_waves)
  int gw_w1 = 0;                 // gate/up tiles of the first wave (= K blocks of the down's first part)
  ActMaps act_k1, act_k2;        // act columns [0, 64 * W1) and [64 * W1, F) as B operands
  int* gw_flag = nullptr;        // gate/up wave 1 passed its PDL wait (epoch)
  unsigned long long* gw_trace = nullptr;  // ECOSERVE_GW_TRACE (debug)
  int gw_epoch = 0;
  float *rope_cos = nullptr, *rope_sin = nullptr;
  int* d_meta = nullptr;
  int* h_meta = nullptr;         // pinned
  int64_t meta_cap = 0;
  int* h_tokens = nullptr;       // pinned [B_max]
  float* dbg = nullptr;          // [(L+1)][T_max][H]
  std::unordered_map<int64_t, std::pair<int, int>> dbg_rows;  // req -> (row0, nrows) of the last phase call
  std::unordered_map<int64_t, Req> reqs;
  Prof prof;
  // decode layer chain (TP=1): per layer the post-attention steps in device memory
  bool chain = false;
  ChainStep* d_chain = nullptr;
  std::vector<int> chain_off, chain_n;
  CUtensorMap* d_amaps = nullptr;            // [3]: h, ao, act as 128-row B operands
  unsigned long long* chain_bar = nullptr;   // grid-barrier counter
  unsigned long long chain_base = 0;
  int* chain_err = nullptr;
  int* h_chain_err = nullptr;                // pinned copy, read after every decode step
  unsigned long long* chain_trace = nullptr;  // ECOSERVE_CHAIN_TRACE=path (debug)
  float* chain_ssp = nullptr;                // [H/128][chain_ss_ld] per-tile sums of squares
  int chain_ss_ld = 0;
  float* chain_ws = nullptr;                 // split-tile sums [1024 tiles][128][128] (zeroed)
  int* chain_cnt = nullptr;                  // [4][1024] tile arrival counters
  double chain_bytes_layer = 0;              // weight bytes streamed per chain launch (O + GU + down + QKV)
  // decode flow (decode_flow.cu): O -> gate/up -> down of a layer as one dataflow kernel
  bool flow = false;
  bool registered = false;                   // counted in device_instances
  float* flow_slots = nullptr;               // [3][num_sms][2][128 * 128] partial tiles
  int* flow_flags = nullptr;                 // [H/128] O flags, then [2F/128] gate/up flags
  int* flow_cnt = nullptr;                   // [6][flow_cnt_ld] arrival + done counters, + [1] down tiles done
  int flow_cnt_ld = 0;
  float* flow_ss = nullptr;                  // [2][H/128][128] sums of squares (after O, after down)
  float* flow_rvec = nullptr;                // [128]
  int* flow_err = nullptr;
  int* h_flow_err = nullptr;                 // pinned copy, read after every decode step
  int flow_epoch = 0;
  unsigned long long* flow_trace = nullptr;  // ECOSERVE_FLOW_TRACE (debug)
  // decode gate/up, stream-K (decode_gu.cu)
  bool gu_sk = false;
  float* gu_part = nullptr;                  // [2F][128] f32 tail partials
  int* gu_flags = nullptr;                   // [2F/128]
  int gu_epoch = 0;
  int* gu_err = nullptr;
  int* h_gu_err = nullptr;                   // pinned copy, read after every decode step
  CUtensorMap gu_actmap, gu_partmap;
  unsigned long long* gu_trace = nullptr;    // ECOSERVE_GU_TRACE (debug)
  int gu_trace_layer = -1;                   // layer being enqueued (trace: layer 5)
  CUtensorMap flow_xmap, flow_actmap;         // x (f32, TMA reduce-add target), act (bf16, TMA store)

  bool fail(const char* what, cudaError_t e) {
    err = std::string(what) + ": " + cudaGetErrorString(e);
    dead = true;
    return false;
  }
};

#define CK(expr)                                                  \
  do {                                                            \
    cudaError_t _e = (expr);                                      \
    if (_e != cudaSuccess) {                                      \
      inst->fail(#expr, _e);                                      \
      return ECOSERVE_ERR_CUDA;                                   \
    }                                                             \
  } while (0)

// TP=2: in-place fp32 sum of the residual stream over the pair (NCCL over NVLink)
#define ALLREDUCE_X(rows)                                                                              \
  do {                                                                                                 \
    if (inst->tp > 1) {                                                                                \
      const int _m = inst->prof.begin(P_OTHER, inst->stream);                                          \
      ncclResult_t _r = ncclAllReduce(inst->x, inst->x, (size_t)(rows) * inst->H, ncclFloat, ncclSum,  \
                                      inst->comm, inst->stream);                                       \
      inst->prof.end(_m, 0, inst->stream);                                                             \
      if (_r != ncclSuccess) {                                                                         \
        inst->err = std::string("ncclAllReduce: ") + ncclGetErrorString(_r);                           \
        inst->dead = true;                                                                             \
        return ECOSERVE_ERR_NCCL;                                                                      \
      }                                                                                                \
    }                                                                                                  \
  } while (0)

// launch `expr` (which launches `nk` kernels) under profiler class `cls` with algorithmic work `w`
#define LAUNCH(cls, w, nk, expr)                                  \
  do {                                                            \
    const int _m = inst->prof.begin((cls), inst->stream);         \
    CK(expr);                                                     \
    inst->prof.end(_m, (w), inst->stream);                        \
    inst->prof.launches += (nk);                                  \
  } while (0)

// The per-rank shape of a TP group (heads and FFN columns are split over
// the tp ranks; hidden size, vocabulary and layer count are not).
static ecoserve_model_shape local_shape(const ecoserve_model_shape* s) {
  ecoserve_model_shape l = *s;
  const int tp = s->tp_size > 0 ? s->tp_size : 1;
  l.n_heads = s->n_heads / tp;
  l.n_kv_heads = s->n_kv_heads / tp;
  l.ffn_dim = s->ffn_dim / tp;
  return l;
}

// Live instances per device. The decode flow kernel's CTAs wait on each other, so they
// must all be resident at once: it only runs while its instance is alone on the GPU
// (another instance's kernels on a concurrent stream could hold SMs indefinitely).
static int device_instances(int device, int delta) {
  static std::mutex mu;
  static std::map<int, int> n;
  std::lock_guard<std::mutex> lock(mu);
  return n[device] += delta;
}

// ECOSERVE_GU_WAVES=1 enables the two-wave decode gate/up with the concurrent first part of
// the down projection (run_layers_decode). Off by default: parity-green and the concurrent
// phase streams at 6.1 TB/s (ECOSERVE_GW_TRACE, tools/gw_trace.py), but the two extra
// kernel boundaries (~3 us TMA ramp after each CTA start + ~3-4 us epilogue tail each) eat
// the gain: 8B B = 128 step 7.91 vs 7.83 ms.
static bool gu_waves_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_GU_WAVES");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// ECOSERVE_PREFILL_DNORM=0: prefill RMSNorms as their own kernels instead of folded into
// the O / down epilogues (h = bf16(x * gamma), per-tile sums of squares) and the QKV /
// gate-up epilogues (x 1/rms) -- A/B measurement.
static bool prefill_dnorm_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_PREFILL_DNORM");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// ECOSERVE_L2_OWN=n: each decode GEMM CTA prefetches up to n of its weight K blocks
// (16 KB each) beyond its smem ring into L2 before its PDL wait (A/B measurement).
static int l2_own_prefetch_kb() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_L2_OWN");
    v = e ? std::max(0, atoi(e)) : 0;
  }
  return v;
}

// ECOSERVE_QKV_FUSE=1: the decode QKV split reduction (RoPE, K/V append) inside the
// attention kernel's prologue instead of its own kernel. Off by default: parity-green but
// measured slower (8B B = 128: 7.93-8.02 vs 7.73-7.80 ms per step) -- the pos -> RoPE
// table round trips delay every attention CTA's first MMA by more than the reduction
// kernel costs.
static bool qkv_fuse_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_QKV_FUSE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// ECOSERVE_FLOW=1 enables the decode flow kernel (decode_flow.cu). Off by default: it is
// parity-green but measured slower than the per-kernel decode path (8B, B = 128, ctx 1.3k:
// 9.09 vs 7.7 ms per decode step).
static bool flow_env_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_FLOW");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// debug: ECOSERVE_FLOW_TRACE=path appends per-CTA phase marks of one flow launch per step
static const char* flow_trace_path() {
  static const char* p = getenv("ECOSERVE_FLOW_TRACE");
  return p;
}

// debug: ECOSERVE_GU_TRACE=path appends per-CTA marks of the gate/up stream-K kernel
// (the launch of layer 5 of each decode step; see tools/flow_trace.py --gu)
static const char* gu_trace_path() {
  static const char* p = getenv("ECOSERVE_GU_TRACE");
  return p;
}

// ECOSERVE_GU_SK=1 enables the stream-K decode gate/up kernel (decode_gu.cu). Off by
// default: parity-green, its mainloop streams at 6.3 TB/s (8B), but the step measured
// slower (8B B = 128: 7.76 vs 7.47 ms; 70B rank shard: 22.5 vs 21.8 ms) -- every CTA now
// ends together, while in the 1.5-wave GEMM the CTAs done after one tile already run
// the down projection's prologue and weight prefetch under PDL.
static bool gu_sk_env_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_GU_SK");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// gate/up flags start on a 128-byte boundary after the O flags (pollers read 16-B vectors)
static int flow_gu_flag_off(int H) { return (H / 128 + 31) / 32 * 32; }

static bool shape_ok(const ecoserve_model_shape* s) {
  if (!s) return false;
  if (s->tp_size != 1 && s->tp_size != 2) return false;
  if (s->n_heads % s->tp_size || s->n_kv_heads % s->tp_size || s->ffn_dim % s->tp_size) return false;
  const ecoserve_model_shape l = local_shape(s);
  if (l.n_layers < 1 || l.hidden < 64 || l.hidden % 64 || l.n_heads < 1 || l.n_kv_heads < 1) return false;
  if (l.n_heads % l.n_kv_heads || l.n_heads / l.n_kv_heads > 16) return false;
  if (!(l.head_dim == 32 || l.head_dim == 64 || l.head_dim == 128)) return false;
  if (l.ffn_dim < 64 || l.ffn_dim % 64 || l.vocab < 1) return false;
  if ((l.n_heads * l.head_dim) % 64) return false;
  return true;
}

namespace {
bool tp_fused_enabled() {  // ECOSERVE_TP_FUSED=0: NCCL all-reduce + separate RMSNorm instead
  const char* e = getenv("ECOSERVE_TP_FUSED");
  return !(e && e[0] == '0');
}

// Exchange the receive buffers of the pair (N2): every rank allocates [2][rows][H]
// receive rows + flags, the pair all-gathers {pid, device, pointers, IPC handles} over
// the NCCL communicator, and maps the peer's buffers -- a direct peer pointer when both
// ranks live in one process, an IPC mapping otherwise.
struct TpPeerInfo {
  int pid, device;
  uint64_t recv, flags;
  cudaIpcMemHandle_t h_recv, h_flags;
};

ecoserve_status tp_setup_peer(ecoserve_instance* inst) {
  inst->tp_rows_max = std::max(inst->T_max, inst->B_max);
  const int64_t rows = inst->tp_rows_max;
  CK(cudaMalloc(&inst->tp_recv, sizeof(float) * 4 * rows * inst->H));
  CK(cudaMalloc(&inst->tp_flags, sizeof(int) * (64 + 2 * rows)));
  CK(cudaMemset(inst->tp_flags, 0, sizeof(int) * (64 + 2 * rows)));
  TpPeerInfo mine{};
  mine.pid = (int)getpid();
  mine.device = inst->device;
  mine.recv = reinterpret_cast<uint64_t>(inst->tp_recv);
  mine.flags = reinterpret_cast<uint64_t>(inst->tp_flags);
  CK(cudaIpcGetMemHandle(&mine.h_recv, inst->tp_recv));
  CK(cudaIpcGetMemHandle(&mine.h_flags, inst->tp_flags));
  void* d_info = nullptr;
  CK(cudaMalloc(&d_info, 2 * sizeof(TpPeerInfo)));
  CK(cudaMemcpy(reinterpret_cast<char*>(d_info) + inst->tp_rank * sizeof(TpPeerInfo), &mine, sizeof(TpPeerInfo),
                cudaMemcpyHostToDevice));
  const ncclResult_t r =
      ncclAllGather(reinterpret_cast<char*>(d_info) + inst->tp_rank * sizeof(TpPeerInfo), d_info, sizeof(TpPeerInfo),
                    ncclChar, inst->comm, inst->stream);
  if (r != ncclSuccess) {
    cudaFree(d_info);
    inst->err = std::string("ncclAllGather: ") + ncclGetErrorString(r);
    return ECOSERVE_ERR_NCCL;
  }
  TpPeerInfo all[2];
  CK(cudaStreamSynchronize(inst->stream));
  CK(cudaMemcpy(all, d_info, sizeof(all), cudaMemcpyDeviceToHost));
  cudaFree(d_info);
  const TpPeerInfo& peer = all[1 - inst->tp_rank];
  if (peer.pid == mine.pid) {
    int ok = 0;
    CK(cudaDeviceCanAccessPeer(&ok, inst->device, peer.device));
    if (!ok) {
      inst->err = "TP pair: no peer access between the two GPUs";
      return ECOSERVE_ERR_CUDA;
    }
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer.device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
    cudaGetLastError();
    inst->peer_recv = reinterpret_cast<float*>(peer.recv);
    inst->peer_flags = reinterpret_cast<int*>(peer.flags);
  } else {
    void* pr = nullptr;
    void* pf = nullptr;
    CK(cudaIpcOpenMemHandle(&pr, peer.h_recv, cudaIpcMemLazyEnablePeerAccess));
    CK(cudaIpcOpenMemHandle(&pf, peer.h_flags, cudaIpcMemLazyEnablePeerAccess));
    inst->peer_recv = reinterpret_cast<float*>(pr);
    inst->peer_flags = reinterpret_cast<int*>(pf);
    inst->peer_ipc = true;
  }
  inst->tp_fused = true;
  return ECOSERVE_OK;
}
}  // namespace

static ecoserve_status build_chain(ecoserve_instance* inst);

extern "C" {

int64_t ecoserve_kv_pool_bytes(const ecoserve_model_shape* s, int32_t block_tokens, int64_t num_blocks) {
  if (!shape_ok(s) || block_tokens != BLOCK || num_blocks < 1) return -1;
  const ecoserve_model_shape l = local_shape(s);
  return num_blocks * (int64_t)l.n_layers * 2 * l.n_kv_heads * BLOCK * l.head_dim * 2;
}

int64_t ecoserve_prepared_weight_bytes(const ecoserve_model_shape* s) {
  if (!shape_ok(s)) return -1;
  const ecoserve_model_shape l = local_shape(s);
  const int64_t qkv = (int64_t)(l.n_heads + 2 * l.n_kv_heads) * l.head_dim * l.hidden;
  const int64_t gu = 2LL * l.ffn_dim * l.hidden;
  return (int64_t)l.n_layers * (qkv + gu) * 2;
}

ecoserve_status ecoserve_nccl_unique_id(void* out) {
  if (!out) return ECOSERVE_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return ECOSERVE_ERR_NCCL;
  memcpy(out, &id, sizeof(id));
  return ECOSERVE_OK;
}

const char* ecoserve_last_error(const ecoserve_instance* inst) { return inst ? inst->err.c_str() : "null instance"; }

static ecoserve_status make_act_maps(ecoserve_instance* inst, ActMaps& m, const void* ptr, int64_t rows, int64_t cols) {
  if (make_tmap_bf16(&m.a, ptr, rows, cols, 128)) return ECOSERVE_ERR_CUDA;
  const int boxes[3] = {64, 128, 256};
  for (int i = 0; i < 3; ++i)
    if (make_tmap_bf16(&m.b[i], ptr, rows, cols, boxes[i])) return ECOSERVE_ERR_CUDA;
  return ECOSERVE_OK;
}

void ecoserve_instance_destroy(ecoserve_instance* inst) {
  if (!inst) return;
  cudaSetDevice(inst->device);
  if (inst->stream) cudaStreamSynchronize(inst->stream);
  void* dev[] = {inst->x, inst->h, inst->q, inst->ao, inst->act, inst->hl, inst->part, inst->counters, inst->attn_ws,
                 inst->am_val,
                 inst->am_idx, inst->d_tokens, inst->sk_cnt, inst->gw_flag, inst->nrm_ss, inst->rope_cos, inst->rope_sin, inst->d_meta, inst->dbg};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (inst->h_meta) cudaFreeHost(inst->h_meta);
  if (inst->h_tokens) cudaFreeHost(inst->h_tokens);
  if (inst->h_chain_err) cudaFreeHost(inst->h_chain_err);
  if (inst->h_tp_err) cudaFreeHost(inst->h_tp_err);
  if (inst->h_flow_err) cudaFreeHost(inst->h_flow_err);
  if (inst->h_gu_err) cudaFreeHost(inst->h_gu_err);
  for (void* p : {(void*)inst->gu_part, (void*)inst->gu_flags, (void*)inst->gu_err, (void*)inst->gu_trace})
    if (p) cudaFree(p);
  for (void* p : {(void*)inst->flow_slots, (void*)inst->flow_flags, (void*)inst->flow_cnt, (void*)inst->flow_ss,
                  (void*)inst->flow_rvec, (void*)inst->flow_err, (void*)inst->flow_trace})
    if (p) cudaFree(p);
  if (inst->registered) device_instances(inst->device, -1);
  if (inst->tp_err) cudaFree(inst->tp_err);
  for (cudaEvent_t e : inst->prof.pool) cudaEventDestroy(e);
  if (inst->peer_ipc) {
    if (inst->peer_recv) cudaIpcCloseMemHandle(inst->peer_recv);
    if (inst->peer_flags) cudaIpcCloseMemHandle(inst->peer_flags);
  }
  for (void* p : {(void*)inst->tp_recv, (void*)inst->tp_flags, (void*)inst->d_wmaps, (void*)inst->d_chain,
                  (void*)inst->d_amaps, (void*)inst->chain_bar, (void*)inst->chain_err, (void*)inst->chain_trace,
                  (void*)inst->chain_ssp, (void*)inst->chain_ws, (void*)inst->chain_cnt})
    if (p) cudaFree(p);
  if (inst->comm) ncclCommDestroy(inst->comm);
  if (inst->own_stream && inst->stream) cudaStreamDestroy(inst->stream);
  delete inst;
}

ecoserve_status ecoserve_instance_create(const ecoserve_model_shape* shape, const ecoserve_kv_pool* kv,
                                         const ecoserve_weights* raw, void* prepared, int32_t device,
                                         int32_t tp_rank, const void* nccl_unique_id, void* cuda_stream,
                                         const ecoserve_engine_config* cfg, ecoserve_instance** out) {
  if (!out) return ECOSERVE_ERR_INVALID_ARG;
  *out = nullptr;
  if (!shape_ok(shape) || !kv || !raw || !prepared || !kv->pool || kv->block_tokens != BLOCK || kv->num_blocks < 1 ||
      !raw->embed || !raw->lm_head || !raw->final_norm || !raw->layers)
    return ECOSERVE_ERR_INVALID_ARG;
  if (shape->tp_size == 1 && (tp_rank != 0 || nccl_unique_id)) return ECOSERVE_ERR_INVALID_ARG;
  if (shape->tp_size == 2 && (tp_rank < 0 || tp_rank > 1 || !nccl_unique_id)) return ECOSERVE_ERR_INVALID_ARG;
  std::unique_ptr<ecoserve_instance> holder(new ecoserve_instance());
  ecoserve_instance* inst = holder.get();
  inst->shape = *shape;
  inst->tp = shape->tp_size;
  inst->tp_rank = tp_rank;
  // every per-head / per-FFN-column dimension below is this rank's shard
  const ecoserve_model_shape ls = local_shape(shape);
  inst->L = ls.n_layers;
  inst->H = ls.hidden;
  inst->M = ls.n_heads;
  inst->Mkv = ls.n_kv_heads;
  inst->D = ls.head_dim;
  inst->F = ls.ffn_dim;
  inst->V = ls.vocab;
  inst->QKV = (inst->M + 2 * inst->Mkv) * inst->D;
  if (cfg) {
    if (cfg->token_budget > 0) inst->T_max = cfg->token_budget;
    if (cfg->max_batch > 0) inst->B_max = cfg->max_batch;
    if (cfg->max_positions > 0) inst->P_max = cfg->max_positions;
    inst->debug = cfg->debug_hidden != 0;
  }
  if (inst->B_max > inst->T_max) inst->T_max = inst->B_max;
  inst->device = device;
  CK(cudaSetDevice(device));
  CK(cudaDeviceGetAttribute(&inst->num_sms, cudaDevAttrMultiProcessorCount, device));
  if (cuda_stream) {
    inst->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  } else {
    CK(cudaStreamCreateWithFlags(&inst->stream, cudaStreamNonBlocking));
    inst->own_stream = true;
  }
  cudaStream_t st = inst->stream;
  const int L = inst->L, H = inst->H, M = inst->M, Mkv = inst->Mkv, D = inst->D, F = inst->F, V = inst->V;
  const int T = inst->T_max;

  // ---- KV pool
  inst->pool = reinterpret_cast<bf16*>(kv->pool);
  inst->num_blocks = kv->num_blocks;
  inst->blk_stride = (int64_t)L * 2 * Mkv * BLOCK * D;
  CK(cudaMemsetAsync(inst->pool, 0, ecoserve_kv_pool_bytes(shape, BLOCK, kv->num_blocks), st));
  inst->free_blocks.resize(kv->num_blocks);
  for (int64_t i = 0; i < kv->num_blocks; ++i) inst->free_blocks[i] = (int)(kv->num_blocks - 1 - i);  // pop_back -> 0,1,..

  // ---- weights: fused + re-laid-out QKV (pair-interleaved q/k rows for RoPE) and gate/up (interleaved)
  inst->embed = reinterpret_cast<const bf16*>(raw->embed);
  inst->lm_head = reinterpret_cast<const bf16*>(raw->lm_head);
  inst->final_norm = reinterpret_cast<const bf16*>(raw->final_norm);
  const int QKV = inst->QKV;
  std::vector<int> sel_qkv(QKV), row_qkv(QKV), sel_gu(2 * F), row_gu(2 * F);
  for (int r = 0; r < QKV; ++r) {
    int base, src_sel;
    if (r < M * D) { base = 0; src_sel = 0; }
    else if (r < (M + Mkv) * D) { base = M * D; src_sel = 1; }
    else { base = (M + Mkv) * D; src_sel = 2; }
    const int rr = r - base;
    sel_qkv[r] = src_sel;
    if (src_sel == 2) {
      row_qkv[r] = rr;
    } else {  // prepared row 2j <- row j, 2j+1 <- row j + D/2 (within a head)
      const int head = rr / D, i = rr % D;
      row_qkv[r] = head * D + ((i & 1) ? i / 2 + D / 2 : i / 2);
    }
  }
  for (int r = 0; r < 2 * F; ++r) { sel_gu[r] = r & 1; row_gu[r] = r / 2; }
  int* d_map = nullptr;
  CK(cudaMalloc(&d_map, sizeof(int) * (2 * QKV + 4 * F)));
  CK(cudaMemcpyAsync(d_map, sel_qkv.data(), sizeof(int) * QKV, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_map + QKV, row_qkv.data(), sizeof(int) * QKV, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_map + 2 * QKV, sel_gu.data(), sizeof(int) * 2 * F, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_map + 2 * QKV + 2 * F, row_gu.data(), sizeof(int) * 2 * F, cudaMemcpyHostToDevice, st));
  bf16* prep = reinterpret_cast<bf16*>(prepared);
  inst->lw.resize(L);
  for (int l = 0; l < L; ++l) {
    const void* const* p = raw->layers + 9 * l;
    for (int i = 0; i < 9; ++i)
      if (!p[i]) return ECOSERVE_ERR_INVALID_ARG;
    LayerW& w = inst->lw[l];
    w.attn_norm = reinterpret_cast<const bf16*>(p[0]);
    w.wo = reinterpret_cast<const bf16*>(p[4]);
    w.ffn_norm = reinterpret_cast<const bf16*>(p[5]);
    w.wd = reinterpret_cast<const bf16*>(p[8]);
    w.wqkv = prep;
    prep += (int64_t)QKV * H;
    w.wgu = prep;
    prep += 2LL * F * H;
    CK(row_gather_launch(reinterpret_cast<const bf16*>(p[1]), reinterpret_cast<const bf16*>(p[2]),
                         reinterpret_cast<const bf16*>(p[3]), d_map, d_map + QKV, w.wqkv, QKV, H, st));
    CK(row_gather_launch(reinterpret_cast<const bf16*>(p[6]), reinterpret_cast<const bf16*>(p[7]), nullptr,
                         d_map + 2 * QKV, d_map + 2 * QKV + 2 * F, w.wgu, 2 * F, H, st));
    if (make_tmap_bf16(&w.qkv_a, w.wqkv, QKV, H, 128) || make_tmap_bf16(&w.qkv_b, w.wqkv, QKV, H, BN_PREFILL) ||
        make_tmap_bf16(&w.o_a, w.wo, H, M * D, 128) || make_tmap_bf16(&w.o_b, w.wo, H, M * D, BN_PREFILL) ||
        make_tmap_bf16(&w.gu_a, w.wgu, 2 * F, H, 128) || make_tmap_bf16(&w.gu_b, w.wgu, 2 * F, H, BN_PREFILL) ||
        make_tmap_bf16(&w.d_a, w.wd, H, F, 128) || make_tmap_bf16(&w.d_b, w.wd, H, F, BN_PREFILL)) {
      inst->err = "cuTensorMapEncodeTiled failed (weights)";
      return ECOSERVE_ERR_CUDA;
    }
  }
  if (make_tmap_bf16(&inst->lm_a, inst->lm_head, V, H, 128)) {
    inst->err = "cuTensorMapEncodeTiled failed (lm_head)";
    return ECOSERVE_ERR_CUDA;
  }
  {  // decode weight maps in global memory for the next-GEMM L2 prefetch
    std::vector<CUtensorMap> maps;
    for (int l = 0; l < L; ++l) {
      const LayerW& w = inst->lw[l];
      maps.push_back(w.qkv_a);
      maps.push_back(w.o_a);
      maps.push_back(w.gu_a);
      maps.push_back(w.d_a);
    }
    maps.push_back(inst->lm_a);
    CK(cudaMalloc(&inst->d_wmaps, sizeof(CUtensorMap) * maps.size()));
    CK(cudaMemcpy(inst->d_wmaps, maps.data(), sizeof(CUtensorMap) * maps.size(), cudaMemcpyHostToDevice));
  }

  // ---- workspace
  CK(cudaMalloc(&inst->x, sizeof(float) * (int64_t)T * H));
  CK(cudaMalloc(&inst->h, 2LL * T * H));
  CK(cudaMalloc(&inst->q, 2LL * T * M * D));
  CK(cudaMalloc(&inst->ao, 2LL * T * M * D));
  CK(cudaMalloc(&inst->act, 2LL * T * F));
  CK(cudaMalloc(&inst->hl, 2LL * inst->B_max * H));
  CK(cudaMemsetAsync(inst->h, 0, 2LL * T * H, st));
  CK(cudaMemsetAsync(inst->ao, 0, 2LL * T * M * D, st));
  CK(cudaMemsetAsync(inst->act, 0, 2LL * T * F, st));
  CK(cudaMemsetAsync(inst->hl, 0, 2LL * inst->B_max * H, st));
  if (make_act_maps(inst, inst->m_h, inst->h, T, H) || make_act_maps(inst, inst->m_ao, inst->ao, T, M * D) ||
      make_act_maps(inst, inst->m_act, inst->act, T, F) || make_act_maps(inst, inst->m_hl, inst->hl, inst->B_max, H)) {
    inst->err = "cuTensorMapEncodeTiled failed (activations)";
    return ECOSERVE_ERR_CUDA;
  }
  {  // tcgen05 prefill attention for head_dim 128 unless ECOSERVE_ATTN_TC=0
    const char* ev = getenv("ECOSERVE_ATTN_TC");
    inst->attn_tc = D == 128 && !(ev && ev[0] == '0');
    const int64_t pool_rows = inst->num_blocks * (int64_t)L * 2 * Mkv * BLOCK;
    if (inst->attn_tc && make_attn_tc_maps(&inst->attn_qmap, &inst->attn_kvmap, inst->q, T, M, inst->pool, pool_rows)) {
      inst->err = "cuTensorMapEncodeTiled failed (attention)";
      return ECOSERVE_ERR_CUDA;
    }
  }
  const int nmax = std::max(QKV, std::max(2 * F, H));
  inst->part_elems = 8LL * inst->B_max * nmax;
  CK(cudaMalloc(&inst->part, sizeof(float) * inst->part_elems));
  CK(cudaMalloc(&inst->counters, sizeof(int) * 16384));
  CK(cudaMemsetAsync(inst->counters, 0, sizeof(int) * 16384, st));
  const int max_blocks_seq = (inst->P_max + BLOCK - 1) / BLOCK;
  inst->attn_ws_elems = (int64_t)inst->B_max * M * 64 * (D + 2);
  CK(cudaMalloc(&inst->attn_ws, sizeof(float) * inst->attn_ws_elems));
  if (gu_waves_enabled() && inst->tp == 1 && F % 64 == 0 && H % 128 == 0 && 2 * F / 128 > inst->num_sms &&
      2 * F / 128 - inst->num_sms <= inst->num_sms - H / 128) {
    // gate/up has more tiles than SMs: W1 = num_sms tiles first, the rest (W2) beside the
    // down projection's K blocks [0, W1) -- those read only first-wave output columns
    const int W1 = inst->num_sms;
    inst->gw_w1 = W1;
    bool bad = false;
    for (int l = 0; l < L && !bad; ++l) {
      LayerW& w = inst->lw[l];
      const int64_t dg[2] = {H, 2LL * F - 128LL * W1}, sg[1] = {2LL * H};
      const int64_t d1[2] = {64LL * W1, H}, d2[2] = {(int64_t)F - 64LL * W1, H}, sd[1] = {2LL * F};
      const int box[2] = {64, 128};
      bad = make_tmap_bf16_nd(&w.gu2_a, w.wgu + 128LL * W1 * H, 2, dg, sg, box) ||
            make_tmap_bf16_nd(&w.d1_a, w.wd, 2, d1, sd, box) ||
            make_tmap_bf16_nd(&w.d2_a, w.wd + 64LL * W1, 2, d2, sd, box);
    }
    for (int i = 0; i < 3 && !bad; ++i) {
      const int boxes[3] = {64, 128, 256};
      const int64_t sa[1] = {2LL * F};
      const int64_t a1[2] = {64LL * W1, T}, a2[2] = {(int64_t)F - 64LL * W1, T};
      const int bx[2] = {64, boxes[i]};
      bad = make_tmap_bf16_nd(&inst->act_k1.b[i], inst->act, 2, a1, sa, bx) ||
            make_tmap_bf16_nd(&inst->act_k2.b[i], inst->act + 64LL * W1, 2, a2, sa, bx);
    }
    if (bad) {
      inst->err = "cuTensorMapEncodeTiled failed (gate/up waves)";
      return ECOSERVE_ERR_CUDA;
    }
    CK(cudaMalloc(&inst->gw_flag, sizeof(int)));
    CK(cudaMemset(inst->gw_flag, 0, sizeof(int)));
  }
  CK(cudaMalloc(&inst->nrm_ss, sizeof(float) * (int64_t)((H + 255) / 256) * T));
  CK(cudaMalloc(&inst->sk_cnt, sizeof(int) * (int64_t)inst->B_max * Mkv));
  CK(cudaMemset(inst->sk_cnt, 0, sizeof(int) * (int64_t)inst->B_max * Mkv));
  inst->am_ld = (V + 127) / 128;
  CK(cudaMalloc(&inst->am_val, sizeof(float) * (int64_t)inst->B_max * inst->am_ld));
  CK(cudaMalloc(&inst->am_idx, sizeof(int) * (int64_t)inst->B_max * inst->am_ld));
  CK(cudaMalloc(&inst->d_tokens, sizeof(int) * inst->B_max));
  inst->meta_cap = 6LL * T + 4 + (int64_t)inst->B_max * (max_blocks_seq + 8) + 2LL * (T / 64 + inst->B_max);
  CK(cudaMalloc(&inst->d_meta, sizeof(int) * inst->meta_cap));
  CK(cudaMallocHost(&inst->h_meta, sizeof(int) * inst->meta_cap));
  CK(cudaMallocHost(&inst->h_tokens, sizeof(int) * inst->B_max));
  // RoPE table: angle(p, i) = p * theta^(-2i/D) in fp64, stored fp32 (reading A3)
  {
    const int half = D / 2;
    std::vector<float> c((int64_t)inst->P_max * half), s((int64_t)inst->P_max * half);
    for (int p = 0; p < inst->P_max; ++p)
      for (int i = 0; i < half; ++i) {
        const double ang = (double)p * pow((double)shape->rope_theta, -2.0 * i / D);
        c[(int64_t)p * half + i] = (float)cos(ang);
        s[(int64_t)p * half + i] = (float)sin(ang);
      }
    CK(cudaMalloc(&inst->rope_cos, sizeof(float) * c.size()));
    CK(cudaMalloc(&inst->rope_sin, sizeof(float) * s.size()));
    CK(cudaMemcpyAsync(inst->rope_cos, c.data(), sizeof(float) * c.size(), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(inst->rope_sin, s.data(), sizeof(float) * s.size(), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  if (inst->debug) CK(cudaMalloc(&inst->dbg, sizeof(float) * (int64_t)(L + 1) * T * H));
  CK(cudaStreamSynchronize(st));
  cudaFree(d_map);
  if (inst->tp > 1) {  // both ranks of the pair call create concurrently (one process per GPU)
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    const ncclResult_t r = ncclCommInitRank(&inst->comm, inst->tp, id, tp_rank);
    if (r != ncclSuccess) {
      inst->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      return ECOSERVE_ERR_NCCL;
    }
    if (tp_fused_enabled()) {
      const ecoserve_status es = tp_setup_peer(inst);
      if (es != ECOSERVE_OK) return es;
      // bound on one exchange wait (the peer may legitimately be a whole prefill GEMM
      // or a host-side hiccup behind); ECOSERVE_TP_TIMEOUT_MS overrides
      const char* e = getenv("ECOSERVE_TP_TIMEOUT_MS");
      inst->tp_timeout_ns = 1000000ull * (unsigned long long)(e ? std::max(1, atoi(e)) : 30000);
      CK(cudaMalloc(&inst->tp_err, sizeof(int)));
      CK(cudaMemset(inst->tp_err, 0, sizeof(int)));
      CK(cudaMallocHost(&inst->h_tp_err, sizeof(int)));
      *inst->h_tp_err = 0;
    }
  }
  if (inst->tp == 1) {
    const ecoserve_status es = build_chain(inst);
    if (es != ECOSERVE_OK) return es;
  }
  if (inst->tp == 1 && !inst->chain && flow_env_enabled() && H % 128 == 0 && F % 64 == 0 && (M * D) % 64 == 0 &&
      2 * F / 128 <= 256 && H / 128 <= 128) {
    const int nt_o = H / 128, nt_gu = 2 * F / 128;
    inst->flow_cnt_ld = std::max(nt_o, nt_gu);
    CK(cudaMalloc(&inst->flow_slots, sizeof(float) * decode_flow_slot_floats(inst->num_sms)));
    CK(cudaMalloc(&inst->flow_flags, sizeof(int) * (flow_gu_flag_off(H) + nt_gu)));  // (128-B aligned groups)
    CK(cudaMemset(inst->flow_flags, 0, sizeof(int) * (flow_gu_flag_off(H) + nt_gu)));
    CK(cudaMalloc(&inst->flow_cnt, sizeof(int) * (6 * inst->flow_cnt_ld + 1)));
    CK(cudaMemset(inst->flow_cnt, 0, sizeof(int) * (6 * inst->flow_cnt_ld + 1)));
    CK(cudaMalloc(&inst->flow_ss, sizeof(float) * 2 * nt_o * 128));
    CK(cudaMalloc(&inst->flow_rvec, sizeof(float) * 128));
    if (flow_trace_path()) {
      CK(cudaMalloc(&inst->flow_trace, sizeof(unsigned long long) * inst->num_sms * 16));
      CK(cudaMemset(inst->flow_trace, 0, sizeof(unsigned long long) * inst->num_sms * 16));
    }
    if (make_tmap_2d_plain(&inst->flow_xmap, inst->x, 1, inst->T_max, H, 128, 32) ||
        make_tmap_2d_plain(&inst->flow_actmap, inst->act, 0, inst->T_max, F, 64, 32)) {
      inst->err = "decode flow: tensor map creation failed";
      return ECOSERVE_ERR_CUDA;
    }
    CK(cudaMalloc(&inst->flow_err, sizeof(int)));
    CK(cudaMemset(inst->flow_err, 0, sizeof(int)));
    CK(cudaMallocHost(&inst->h_flow_err, sizeof(int)));
    *inst->h_flow_err = 0;
    inst->flow = true;
  }
  if (gu_sk_env_enabled() && F % 64 == 0 && H % 64 == 0) {
    CK(cudaMalloc(&inst->gu_part, sizeof(float) * 2LL * F * 128));
    CK(cudaMalloc(&inst->gu_flags, sizeof(int) * (2 * F / 128 + 1)));
    CK(cudaMemset(inst->gu_flags, 0, sizeof(int) * (2 * F / 128 + 1)));
    CK(cudaMalloc(&inst->gu_err, sizeof(int)));
    CK(cudaMemset(inst->gu_err, 0, sizeof(int)));
    CK(cudaMallocHost(&inst->h_gu_err, sizeof(int)));
    *inst->h_gu_err = 0;
    if (make_tmap_2d_plain(&inst->gu_actmap, inst->act, 0, inst->T_max, F, 64, 32) ||
        make_tmap_2d_plain(&inst->gu_partmap, inst->gu_part, 1, 2LL * F, 128, 128, 32)) {
      inst->err = "gate/up stream-K: tensor map creation failed";
      return ECOSERVE_ERR_CUDA;
    }
    inst->gu_sk = true;
  }
  device_instances(device, +1);  // (a failed create is not counted)
  inst->registered = true;
  *out = holder.release();
  return ECOSERVE_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ forward
namespace {

struct LayerIO {
  int rows;          // tokens in this batch
  const int* pos;    // device
  const int* slot;   // device
};

static bool epi_bulk_enabled() {  // ECOSERVE_EPI_BULK=1: GemmEpi::bulk_copy
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_EPI_BULK");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

GemmEpi epi_base(ecoserve_instance* inst) {
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.bulk_copy = epi_bulk_enabled() ? 1 : 0;
  e.rope_cos = inst->rope_cos;
  e.rope_sin = inst->rope_sin;
  e.indep = 2;  // prefill: the weights are the B operand
  e.n_heads = inst->M;
  e.n_kv = inst->Mkv;
  e.head_dim = inst->D;
  e.blk_stride = inst->blk_stride;
  e.q_out = inst->q;
  return e;
}

// Residual update after the O / down projection. TP=1: x += acc. TP=2 (row a17,
// P:276-283): rank 0 writes x + acc_0, rank 1 writes acc_1, and one NCCL all-reduce
// (sum, fp32, in place) forms x + acc_0 + acc_1 -- bitwise identical on both ranks,
// so the replicated LM head takes the same argmax without another collective.
GemmEpi resid_epi(ecoserve_instance* inst) {
  GemmEpi e = epi_base(inst);
  e.resid = inst->x;
  e.ldr = inst->H;
  e.out = inst->x;
  e.ldo = inst->H;
  return e;
}
int resid_mode_prefill(const ecoserve_instance* inst) { return inst->tp_rank == 0 ? EPI_RESID : EPI_F32; }
int resid_mode_decode(const ecoserve_instance* inst) { return inst->tp_rank == 0 ? EPI_SWAP_RESID : EPI_SWAP_STORE; }

bf16* k_layer(ecoserve_instance* inst, int l) { return inst->pool + (int64_t)l * 2 * inst->Mkv * BLOCK * inst->D; }
bf16* v_layer(ecoserve_instance* inst, int l) { return k_layer(inst, l) + (int64_t)inst->Mkv * BLOCK * inst->D; }

bool chain_enabled() {  // ECOSERVE_CHAIN=1: the decode layer chain (work in progress: off by default)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_CHAIN");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

}  // namespace

// The decode layer chain (kernels.h ChainStep) of every layer, built once: after the
// attention of layer l, one persistent kernel runs the GEMMs
//   O (x += o Wo^T; hb = bf16(x * ffn_norm); sum of squares per token and 128-feature tile)
//   gate/up (x the RMSNorm scale r per token; SiLU * up)
//   down (x += ...; hb = bf16(x * attn_norm(l+1)) -- the last layer: final_norm into hl)
//   QKV of layer l+1 (x r; RoPE, q, paged K / V)
// The RMSNorm is split around the GEMM: gamma is applied to the GEMM input, 1/rms to its
// output (sum_k bf16(x_k gamma_k) W_jk * r instead of sum_k bf16(x_k r gamma_k) W_jk,
// the same bf16 rounding per element). The LM head reads bf16(x * final_norm): argmax
// is invariant to the positive per-token scale r.
static ecoserve_status build_chain(ecoserve_instance* inst) {
  const int L = inst->L, H = inst->H, M = inst->M, D = inst->D, F = inst->F, QKV = inst->QKV;
  inst->chain = false;
  if (!chain_enabled() || H % 128 || (2 * F) % 128 || QKV % 128 || (M * D) % 64 || F % 64 || inst->B_max > 512)
    return ECOSERVE_OK;
  {
    CUtensorMap am[3] = {inst->m_h.b[1], inst->m_ao.b[1], inst->m_act.b[1]};
    CK(cudaMalloc(&inst->d_amaps, sizeof(am)));
    CK(cudaMemcpy(inst->d_amaps, am, sizeof(am), cudaMemcpyHostToDevice));
  }
  inst->chain_ss_ld = inst->B_max;
  CK(cudaMalloc(&inst->chain_ssp, sizeof(float) * (H / 128) * inst->chain_ss_ld));
  CK(cudaMalloc(&inst->chain_ws, sizeof(float) * 1024LL * 128 * 128));
  CK(cudaMemset(inst->chain_ws, 0, sizeof(float) * 1024LL * 128 * 128));
  CK(cudaMalloc(&inst->chain_cnt, sizeof(int) * 4 * 1024));
  CK(cudaMemset(inst->chain_cnt, 0, sizeof(int) * 4 * 1024));
  const int max_tiles = ((std::max(std::max(2 * F, QKV), H) + 127) / 128) * ((inst->B_max + 127) / 128);
  if (max_tiles > 1024) return ECOSERVE_OK;
  std::vector<ChainStep> steps;
  auto gemm = [&](int map_idx, int amap, int m_rows, int K, int mode) -> ChainStep& {
    ChainStep c;
    memset(&c, 0, sizeof(c));
    c.wmap = inst->d_wmaps + map_idx;
    c.xmap = inst->d_amaps + amap;
    c.m_rows = m_rows;
    c.K = K;
    c.mode = mode;
    c.H = H;
    c.eps = inst->shape.rms_eps;
    c.ssp_tiles = H / 128;
    c.counters = inst->chain_cnt + 1024 * (int)(steps.size() % 4);
    steps.push_back(c);
    return steps.back();
  };
  inst->chain_off.assign(L, 0);
  inst->chain_n.assign(L, 0);
  for (int l = 0; l < L; ++l) {
    const LayerW& w = inst->lw[l];
    const bool last = l + 1 == L;
    inst->chain_off[l] = (int)steps.size();
    {
      ChainStep& c = gemm(4 * l + 1, 1, H, M * D, CE_RESID_SS);
      c.x = inst->x;
      c.gamma = w.ffn_norm;
      c.hb = inst->h;
      c.ssp_out = inst->chain_ssp;
    }
    {
      ChainStep& c = gemm(4 * l + 2, 0, 2 * F, H, CE_SILU_R);
      c.ssp_in = inst->chain_ssp;
      c.e = epi_base(inst);
      c.e.out = inst->act;
      c.e.ldo = F;
    }
    {
      ChainStep& c = gemm(4 * l + 3, 2, H, F, CE_RESID_SS);
      c.x = inst->x;
      c.gamma = last ? inst->final_norm : inst->lw[l + 1].attn_norm;
      c.hb = last ? inst->hl : inst->h;
      c.ssp_out = inst->chain_ssp;
    }
    if (!last) {
      ChainStep& c = gemm(4 * (l + 1), 0, QKV, H, CE_QKV_R);
      c.ssp_in = inst->chain_ssp;
      c.e = epi_base(inst);
      c.e.k_cache = k_layer(inst, l + 1);
      c.e.v_cache = v_layer(inst, l + 1);
    }
    inst->chain_n[l] = (int)steps.size() - inst->chain_off[l];
  }
  CK(cudaMalloc(&inst->d_chain, sizeof(ChainStep) * steps.size()));
  CK(cudaMemcpy(inst->d_chain, steps.data(), sizeof(ChainStep) * steps.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&inst->chain_bar, sizeof(unsigned long long)));
  CK(cudaMemset(inst->chain_bar, 0, sizeof(unsigned long long)));
  CK(cudaMalloc(&inst->chain_err, sizeof(int)));
  CK(cudaMemset(inst->chain_err, 0, sizeof(int)));
  CK(cudaMallocHost(&inst->h_chain_err, sizeof(int)));
  *inst->h_chain_err = 0;
  inst->chain_base = 0;
  inst->chain_bytes_layer = 2.0 * ((double)H * M * D + 2.0 * F * H + (double)H * F + (double)QKV * H);
  inst->chain = true;
  return ECOSERVE_OK;
}

namespace {

// Prefill projection: CTA-pair 256 x 256 tiles (cta_group::2) unless ECOSERVE_GEMM2=0,
// then the 1-CTA 128 x 256 kernel. w128 / w256: the weight's tensor maps with 128 / 256-row boxes.
bool use_gemm2() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_GEMM2");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

cudaError_t prefill_gemm(ecoserve_instance* inst, const CUtensorMap& amap, const CUtensorMap& w128,
                         const CUtensorMap& w256, int T, int N, int K, const GemmEpi& e) {
  if (use_gemm2()) return gemm2_launch(&amap, &w128, T, N, K, e, inst->num_sms, inst->stream);
  return gemm_launch(&amap, &w256, T, N, K, BN_PREFILL, 1, e, inst->num_sms, inst->stream);
}

// Skinny decode GEMM (swap-AB): weights on the MMA M side, the B tokens on N, K split so
// the grid fills the SMs; the epilogue (and the split reduction) run inside the kernel.
int decode_variant() {  // 1: one A+B ring (default); 3: lean (co-resident); 4: split weight / activation rings
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_DEC_VARIANT");
    v = e ? atoi(e) : 1;
    if (v != 1 && v != 3 && v != 4) v = 1;
  }
  return v;
}

// Off by default: standalone the cluster kernel beats partials + reduction (O 12.8 vs
// 11.5 + 7 us), but inside the decode step it measured 15-20 us slower per launch
// (bench r01: decode 11.7k vs 13.8k tok/s) -- clusters need whole free GPC slices, so
// they cannot start while the previous kernel's CTAs drain under PDL.
// ECOSERVE_CLUSTER_SPLITK=1 enables it.
// Timing experiments only (tools/decode_ablate.py): ECOSERVE_ABLATE=<bitmask> drops
// kernels from the decode step so their in-step cost can be measured by difference:
// 1 = decode attention, 2 = O / gate-up / down GEMMs and their reductions, 4 = the QKV
// GEMM. The tokens are then meaningless; never set in the product path.
int ablate_mask() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_ABLATE");
    v = e ? atoi(e) : 0;
  }
  return v;
}

bool host_timing_enabled() {  // ECOSERVE_HOST_TIMING=1: per decode step host-enqueue vs wall time (stderr)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_HOST_TIMING");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool use_cluster_splitk() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_CLUSTER_SPLITK");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Next-GEMM L2 prefetch (ECOSERVE_L2_PREFETCH=1): measured neutral in the bench step
// (decode 14.74k vs 14.81k tok/s on one box) -- the next kernel's pre-PDL-wait weight
// loads already cover the boundary -- so off by default.
bool use_l2_prefetch() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_L2_PREFETCH");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// The next decode GEMM (weights `map_idx` in d_wmaps, n_out x K) as the L2-prefetch
// target of the current one.
void set_prefetch(ecoserve_instance* inst, GemmEpi& e, int map_idx, int n_out, int K, int B) {
  if (!use_l2_prefetch()) return;
  const int bn = B <= 64 ? 64 : 128;
  e.pf_map = inst->d_wmaps + map_idx;
  e.pf_m_rows = n_out;
  e.pf_K = K;
  e.pf_splits = gemm_effective_splits(K, gemm_decode_splits(n_out, K, inst->num_sms));
  e.pf_n_tiles = (B + bn - 1) / bn;
  e.pf_kb = 6;
}

// norm_gamma / norm_out (optional): when the projection is a residual add split over K,
// its reduction is fused with the following RMSNorm (one kernel: x += sum of partials,
// out = rmsnorm(x) * gamma); *fused reports whether that happened.
// ECOSERVE_PAIR_TILES=1: gate/up decode GEMM with two 128-row weight tiles per CTA (one wave
// of 112 CTAs for 224 tiles) instead of one tile per CTA (148 + 76); measured neutral
// (8B decode 15.36k vs 15.46k tok/s, 70B shard 20.99 vs 21.16 ms/step), so off by default
bool pair_tiles_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_PAIR_TILES");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// ECOSERVE_DEC_R2=1: every decode projection streams two 128-row weight tiles per work
// unit behind one activation tile (256-row weight box). The TMA probe
// (profiles/r01_tma_stream_probe.jsonl) caps one SM's TMA streaming at ~94 GB/s; with
// one weight and one activation tile per stage only half of it is weights, with two
// weight tiles two thirds. Splits are re-chosen for 256-row units (up to 8).
bool dec_r2_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_DEC_R2");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int decode_splits_r2(int n_out, int K, int num_sms) {
  const int units = (n_out + 255) / 256;
  if (4 * units >= 3 * num_sms) return 1;
  const int kb_total = (K + 63) / 64;
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= 8; ++s) {
    const int eff = gemm_effective_splits(K, s);
    if (eff != s) continue;
    const int kb_per = (kb_total + eff - 1) / eff;
    const int waves = (units * eff + num_sms - 1) / num_sms;
    const double cost = (double)waves * kb_per * 2 + (eff > 1 ? 0.5 * eff : 0.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = eff;
    }
  }
  return best;
}

unsigned long long* gu_trace_buf(ecoserve_instance* inst) {
  if (!gu_trace_path() || inst->gu_trace_layer != 5) return nullptr;
  if (!inst->gu_trace) {
    if (cudaMalloc(&inst->gu_trace, sizeof(unsigned long long) * inst->num_sms * 16) != cudaSuccess) return nullptr;
    cudaMemset(inst->gu_trace, 0, sizeof(unsigned long long) * inst->num_sms * 16);
  }
  return inst->gu_trace;
}

bool qkv_inkernel_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_QKV_INKERNEL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// ECOSERVE_DEC_SK=1: the split decode projections (O, down, QKV when their weight tiles
// are fewer than the SMs) use the balanced split (GemmEpi::sk_L) instead of a uniform one
bool dec_sk_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_DEC_SK");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Chunk length of the balanced split of an n_out x K decode projection (0 = use the
// uniform split): one token tile, at most 8 partial slots per tile (inst->part holds 8
// planes of B_max x the widest split output).
int balanced_chunk(ecoserve_instance* inst, int n_out, int K, int B) {
  const int bn = B <= 64 ? 64 : 128;
  if (!dec_sk_enabled() || B > bn) return 0;
  return gemm_sk_chunk((n_out + 127) / 128, (K + 63) / 64, inst->num_sms, 8);
}

cudaError_t decode_gemm(ecoserve_instance* inst, const CUtensorMap& wmap, const ActMaps& xm, int n_out, int K, int B,
                        int mode, GemmEpi e, int* nk, const bf16* norm_gamma = nullptr, bf16* norm_out = nullptr,
                        bool* fused = nullptr, const CUtensorMap* wmap256 = nullptr) {
  const int bn = B <= 64 ? 64 : 128;  // B > 128: several 128-token tiles; weight re-reads hit L2
  const bool r2 = wmap256 && dec_r2_enabled() && (B + bn - 1) / bn == 1 && n_out >= 256;
  const int splits = r2 ? decode_splits_r2(n_out, K, inst->num_sms) : gemm_decode_splits(n_out, K, inst->num_sms);
  const CUtensorMap* wm = r2 ? wmap256 : &wmap;
  const int rr = r2 ? 2 : decode_variant();
  const int var = rr;
  if (fused) *fused = false;
  e.indep = 1;  // weights (A) prefetch before the PDL wait
  e.l2_pf_kb = l2_own_prefetch_kb();
  if (r2) e.pf_map = nullptr;  // (the L2 prefetch assumes 128-row units)
  if (splits == 1 && r2) {
    e.mode = mode;
    *nk = 1;
    return gemm_launch_r(wm, &xm.b[bn_index(bn)], n_out, B, K, bn, 2, 1, e, inst->num_sms, inst->stream);
  }
  if (splits == 1 && mode == EPI_SWAP_SILU && inst->gu_sk && gu_sk_applicable(n_out, K, B, inst->num_sms) &&
      device_instances(inst->device, 0) == 1) {
    // more weight tiles than SMs: balanced stream-K with deterministic two-way tile sums
    // (decode_gu.cu); its CTAs wait on each other, so only while alone on the GPU
    GuSkArgs ga;
    ga.m_rows = n_out;
    ga.K = K;
    ga.B = B;
    ga.epoch = ++inst->gu_epoch;
    ga.flags = inst->gu_flags;
    ga.err = inst->gu_err;
    ga.trace = gu_trace_buf(inst);
    *nk = 1;
    return gu_sk_launch(&wmap, &xm.b[bn_index(bn)], &inst->gu_actmap, &inst->gu_partmap, ga, bn, inst->num_sms,
                        inst->stream);
  }
  if (splits == 1) {  // epilogue in the GEMM
    e.mode = mode;
    *nk = 1;
    const int tiles = (n_out + 127) / 128;
    // more tiles than SMs: two weight tiles (a 256-row box) per CTA behind one activation
    // tile, so all units run in one wave (gate/up: 112 units instead of 148 + 76)
    if (wmap256 && mode == EPI_SWAP_SILU && pair_tiles_enabled() && tiles > inst->num_sms &&
        (tiles + 1) / 2 <= inst->num_sms && (B + bn - 1) / bn == 1)
      return gemm_launch_r(wmap256, &xm.b[bn_index(bn)], n_out, B, K, bn, 2, 1, e, inst->num_sms, inst->stream);
    return gemm_launch_r(&wmap, &xm.b[bn_index(bn)], n_out, B, K, bn, var, 1, e, inst->num_sms, inst->stream);
  }
  // split-K over a thread-block cluster, reduced in distributed shared memory with the
  // epilogue in the same kernel (no partials in HBM; ECOSERVE_CLUSTER_SPLITK=0 disables)
  if (use_cluster_splitk() && splits <= 4) {
    // fewer splits when the clusters of `splits` CTAs would not all be resident at once
    const int tiles = ((n_out + 127) / 128) * ((B + bn - 1) / bn);
    int sc = splits;
    while (sc >= 2 && gemm_cluster_max_active(bn, sc) < tiles) --sc;
    sc = sc >= 2 ? gemm_effective_splits(K, sc) : 0;
    if (sc >= 2) {
      e.mode = mode;
      *nk = 1;
      return gemm_cluster_launch(&wmap, &xm.b[bn_index(bn)], n_out, B, K, bn, sc, e, inst->stream);
    }
  }
  // ECOSERVE_QKV_INKERNEL=1: the QKV split reduction (+ RoPE, K/V append) by the last CTA
  // of each weight tile inside the GEMM (GemmEpi::part / counters) instead of a reduction kernel
  if (mode == EPI_SWAP_QKV && qkv_inkernel_enabled() && var == 1 && !r2 && (B + bn - 1) / bn == 1) {
    e.mode = mode;
    e.part = inst->part;
    e.counters = inst->counters;
    *nk = 1;
    return gemm_launch_r(&wmap, &xm.b[bn_index(bn)], n_out, B, K, bn, 1, splits, e, inst->num_sms, inst->stream);
  }
  // split-K: f32 partials, then one fixed-order reduction kernel applying the epilogue
  GemmEpi ge = e;
  ge.mode = EPI_SWAP_F32;
  ge.out = inst->part;
  ge.ldo = n_out;
  int sk_L = 0;
  if (!r2 && var == 1) sk_L = balanced_chunk(inst, n_out, K, B);
  if (sk_L > 0) {  // balanced split: equal K-block chunks on every SM
    ge.sk_L = e.sk_L = sk_L;
    ge.sk_kbt = e.sk_kbt = (K + 63) / 64;
  }
  cudaError_t r = gemm_launch_r(wm, &xm.b[bn_index(bn)], n_out, B, K, bn, var, sk_L > 0 ? 1 : splits, ge,
                                inst->num_sms, inst->stream);
  if (r != cudaSuccess) return r;
  if (norm_gamma && mode == EPI_SWAP_RESID && n_out == inst->H) {
    *nk = 2;
    if (fused) *fused = true;
    return splitk_resid_rmsnorm_launch(inst->part, splits, B, inst->x, norm_gamma, norm_out, inst->H,
                                       inst->shape.rms_eps, inst->stream, ge.sk_L, ge.sk_kbt);
  }
  const int red = mode == EPI_SWAP_QKV ? RED_QKV : mode == EPI_SWAP_SILU ? RED_SILU
                : mode == EPI_SWAP_RESID ? RED_RESID : mode == EPI_SWAP_STORE ? RED_F32 : RED_BF16;
  *nk = 2;
  return splitk_reduce_launch(red, inst->part, splits, B, n_out, n_out, e, inst->stream);
}

// TP=2 fused path (N2): the receive plane of rank `r` for the exchange of epoch `ep`
// on this GPU (mine) or on the peer (over NVLink).
float* tp_plane(ecoserve_instance* inst, bool peer, int ep, int r) {
  float* base = peer ? inst->peer_recv : inst->tp_recv;
  return base + ((int64_t)(ep & 1) * 2 + r) * inst->tp_rows_max * inst->H;
}

// The epilogue of an O / down projection of a TP rank: its f32 output goes to its own
// receive plane here and, tile by tile while the GEMM runs, to the peer's (out2).
GemmEpi tp_push_epi(ecoserve_instance* inst, int ep) {
  GemmEpi e = epi_base(inst);
  e.out = tp_plane(inst, false, ep, inst->tp_rank);
  e.resid = reinterpret_cast<float*>(e.out);
  e.ldo = e.ldr = inst->H;
  e.out2 = tp_plane(inst, true, ep, inst->tp_rank);
  return e;
}

// Decode O / down projection of a TP rank: raw f32 split partials [splits][B][n_out] in
// inst->part (bulk-stored, L2-resident), summed and pushed row by row by tp_push_rows.
// sk (optional): the balanced split's chunk / K blocks when it was used (sk[0] = 0 otherwise)
cudaError_t decode_partials(ecoserve_instance* inst, const CUtensorMap& wmap, const ActMaps& xm, int n_out, int K,
                            int B, int* splits_out, int* sk = nullptr) {
  const int bn = B <= 64 ? 64 : 128;
  const int splits = gemm_effective_splits(K, gemm_decode_splits(n_out, K, inst->num_sms));
  GemmEpi ge = epi_base(inst);
  ge.mode = EPI_SWAP_F32;
  ge.out = inst->part;
  ge.ldo = n_out;
  ge.indep = 1;
  *splits_out = splits;
  const int var = decode_variant();
  const int L = (sk && splits > 1 && var == 1) ? balanced_chunk(inst, n_out, K, B) : 0;
  if (sk) {
    sk[0] = L;
    sk[1] = (K + 63) / 64;
  }
  if (L > 0) {
    ge.sk_L = L;
    ge.sk_kbt = (K + 63) / 64;
  }
  return gemm_launch_r(&wmap, &xm.b[bn_index(bn)], n_out, B, K, bn, var, L > 0 ? 1 : splits, ge, inst->num_sms,
                       inst->stream);
}

// Decode O / down projection of a TP rank whose bulk f32 epilogue writes its split
// partials [splits][B][H] both to this GPU's receive plane and, over NVLink, to the
// peer's; tp_allreduce then sums both ranks' partials locally (same order and bits as
// the per-row push). Measured slower than the per-row push (70B TP=2 decode 26.0 vs
// 25.0 ms/step: the remote stores stretch the GEMM's tail), so ECOSERVE_TP_DECODE_PUSH=1
// opts in.
bool tp_decode_push_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ECOSERVE_TP_DECODE_PUSH");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

cudaError_t decode_partials_push(ecoserve_instance* inst, const CUtensorMap& wmap, const ActMaps& xm, int n_out, int K,
                                 int B, int ep, int* splits_out) {
  const int bn = B <= 64 ? 64 : 128;
  const int splits = gemm_effective_splits(K, gemm_decode_splits(n_out, K, inst->num_sms));
  GemmEpi ge = epi_base(inst);
  ge.mode = EPI_SWAP_F32;
  ge.out = tp_plane(inst, false, ep, inst->tp_rank);
  ge.out2 = tp_plane(inst, true, ep, inst->tp_rank);
  ge.ldo = n_out;
  ge.indep = 1;
  *splits_out = splits;
  return gemm_launch_r(&wmap, &xm.b[bn_index(bn)], n_out, B, K, bn, 1, splits, ge, inst->num_sms, inst->stream);
}

cudaError_t tp_push_rows(ecoserve_instance* inst, int ep, int splits, int rows, const bf16* gamma, bf16* h,
                         const int* sk = nullptr) {
  TpRowsArgs a;
  a.sk_L = sk ? sk[0] : 0;
  a.sk_kbt = sk ? sk[1] : 0;
  a.part = inst->part;
  a.splits = splits;
  a.plane = (int64_t)rows * inst->H;
  a.ldp = inst->H;
  a.x = inst->x;
  a.gamma = gamma;
  a.h = h;
  a.eps = inst->shape.rms_eps;
  a.rows = rows;
  a.H = inst->H;
  a.rank = inst->tp_rank;
  a.epoch = ep;
  a.peer_recv = tp_plane(inst, true, ep, 0);
  a.my_recv = tp_plane(inst, false, ep, 0);
  a.peer_flags = inst->peer_flags + 64 + (ep & 1) * inst->tp_rows_max;
  a.my_flags = inst->tp_flags + 64 + (ep & 1) * inst->tp_rows_max;
  a.err = inst->tp_err;
  a.timeout_ns = inst->tp_timeout_ns;
  return tp_push_rows_launch(a, inst->num_sms, inst->stream);
}

// After the push GEMM of epoch `ep`: wait for the peer's push, x = (x + acc_0) + acc_1,
// and the next RMSNorm (gamma null: x only).
cudaError_t tp_allreduce(ecoserve_instance* inst, int ep, int rows, const bf16* gamma, bf16* h, int splits = 1) {
  TpAllreduceArgs a;
  a.recv0 = tp_plane(inst, false, ep, 0);
  a.recv1 = tp_plane(inst, false, ep, 1);
  a.splits = splits;
  a.x = inst->x;
  a.gamma = gamma;
  a.h = h;
  a.eps = inst->shape.rms_eps;
  a.rows = rows;
  a.H = inst->H;
  a.epoch = ep;
  a.peer_flag = inst->peer_flags;
  a.my_flag = inst->tp_flags;
  a.err = inst->tp_err;
  a.timeout_ns = inst->tp_timeout_ns;
  return tp_allreduce_norm_launch(a, inst->num_sms, inst->stream);
}

}  // namespace

// The decode flow kernel runs when the instance set it up (TP=1, ECOSERVE_FLOW=1),
// the batch fits one 128-token tile and the instance is alone on its GPU (device_instances).
static bool use_flow(ecoserve_instance* inst, int B) {
  return inst->flow && B >= 1 && B <= 128 && device_instances(inst->device, 0) == 1;
}

// Context splits of the decode attention: split only as much as needed for
// B x Mkv x splits to fill the SMs about twice (uniform 512-token chunks were measured
// slower: more CTAs, partials, combine). ECOSERVE_ATTN_SPLITS=n forces n (sweeps).
static int decode_attn_splits(const ecoserve_instance* inst, int B, int max_blocks, int* bps) {
  static int forced = -1;
  if (forced < 0) {
    const char* e = getenv("ECOSERVE_ATTN_SPLITS");
    forced = e ? std::max(0, atoi(e)) : 0;
  }
  int n = forced > 0 ? forced : std::max(1, (2 * inst->num_sms + B * inst->Mkv - 1) / (B * inst->Mkv));
  n = std::max(1, std::min(std::min(n, max_blocks), 64));
  *bps = (max_blocks + n - 1) / n;
  return (max_blocks + *bps - 1) / *bps;
}

// Hybrid (chunked-prefill + decode) batch of ecoserve_hybrid_step: rows [0, Tc) are
// prompt chunks (prefill attention with per-chunk context offsets), rows [Tc, Tc + n_dec)
// one decode token each (split-K decode attention over the pool).
struct HybridTail {
  int Tc = 0;
  const int* d_ctx_off = nullptr;  // [n_chunks]
  int n_dec = 0;
  const int* d_ctx = nullptr;      // [n_dec] context incl. the current token
  const int* d_bt = nullptr;       // [n_dec][bt_ld]
  int bt_ld = 1;
  const int* d_order = nullptr;    // [n_dec] longest context first
  int n_splits = 1, bps = 1;
  double kv_bytes = 0;
};

static ecoserve_status run_layers_prefill(ecoserve_instance* inst, int T, const int* d_ids, const int* d_pos,
                                          const int* d_slot, const int* d_cu, const int* d_bt, int bt_ld,
                                          const int* d_tiles, int n_tiles, double attn_flop,
                                          const HybridTail* hy = nullptr) {
  cudaStream_t st = inst->stream;
  const int L = inst->L, H = inst->H, M = inst->M, D = inst->D, F = inst->F;
  const float eps = inst->shape.rms_eps;
  LAUNCH(P_OTHER, 0, 1, embed_launch(d_ids, inst->embed, inst->x, T, H, inst->V, st));
  if (inst->debug) CK(cudaMemcpyAsync(inst->dbg, inst->x, sizeof(float) * (int64_t)T * H, cudaMemcpyDeviceToDevice, st));
  bool h_ready = false;  // the previous layer's fused TP all-reduce already wrote this layer's norm
  // deferred RMSNorm (TP=1): the residual epilogues leave h = bf16(x * gamma) and per-tile
  // sums of x^2, the consumer epilogues multiply by 1/rms (GemmEpi::nrm_*)
  const bool dnorm = inst->tp == 1 && prefill_dnorm_enabled();
  bool ss_ready = false;  // h is bf16(x * gamma) and nrm_ss holds the row sums: consumers scale
  auto nrm_in = [&](GemmEpi& g) {
    if (!ss_ready) return;
    g.nrm_ss_in = inst->nrm_ss;
    g.nrm_ss_ld = inst->T_max;
    g.nrm_ss_n = (H + 255) / 256;
    g.nrm_inv_h = 1.f / (float)H;
    g.nrm_eps = eps;
  };
  auto nrm_out = [&](GemmEpi& g, const bf16* gamma) {
    g.nrm_h = inst->h;
    g.nrm_ldh = H;
    g.nrm_gamma = gamma;
    g.nrm_ss_out = inst->nrm_ss;
    g.nrm_ss_ld = inst->T_max;
  };
  for (int l = 0; l < L; ++l) {
    LayerW& w = inst->lw[l];
    if (!h_ready) LAUNCH(P_OTHER, 0, 1, rmsnorm_launch(inst->x, H, nullptr, w.attn_norm, inst->h, T, H, eps, st));
    h_ready = false;
    GemmEpi e = epi_base(inst);
    nrm_in(e);
    ss_ready = false;
    e.mode = EPI_QKV;
    e.pos = d_pos;
    e.slot = d_slot;
    e.k_cache = k_layer(inst, l);
    e.v_cache = v_layer(inst, l);
    LAUNCH(P_GEMM_PREFILL, 2.0 * T * inst->QKV * H, 1,
           prefill_gemm(inst, inst->m_h.a, w.qkv_a, w.qkv_b, T, inst->QKV, H, e));
    PrefillAttnArgs a;
    a.q = inst->q;
    a.k_cache = k_layer(inst, l);
    a.v_cache = v_layer(inst, l);
    a.blk_stride = inst->blk_stride;
    a.cu_seqlens = d_cu;
    a.block_tables = d_bt;
    a.bt_ld = bt_ld;
    a.tiles = d_tiles;
    a.ctx_off = hy ? hy->d_ctx_off : nullptr;
    a.n_tiles = n_tiles;
    a.out = inst->ao;
    a.n_heads = M;
    a.n_kv = inst->Mkv;
    a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
    if (n_tiles > 0) {
      if (inst->attn_tc)
        LAUNCH(P_ATTN_PREFILL, attn_flop, 1,
               attn_prefill_tc_launch(&inst->attn_qmap, &inst->attn_kvmap, d_cu, d_bt, bt_ld, d_tiles, n_tiles,
                                      inst->ao, M, inst->Mkv, l, inst->L, st, a.ctx_off,
                                      (int)(attn_flop / (4.0 * M * D * std::max(1, T)))));
      else
        LAUNCH(P_ATTN_PREFILL, attn_flop, 1, attn_prefill_launch(a, D, st));
    }
    if (hy && hy->n_dec > 0) {  // decode rows of a hybrid batch
      DecodeAttnArgs da;
      da.q = inst->q + (int64_t)hy->Tc * M * D;
      da.k_cache = k_layer(inst, l);
      da.v_cache = v_layer(inst, l);
      da.blk_stride = inst->blk_stride;
      da.ctx_lens = hy->d_ctx;
      da.block_tables = hy->d_bt;
      da.bt_ld = hy->bt_ld;
      da.B = hy->n_dec;
      da.n_heads = M;
      da.n_kv = inst->Mkv;
      da.n_splits = hy->n_splits;
      da.blocks_per_split = hy->bps;
      da.part_o = inst->attn_ws;
      da.part_ml = inst->attn_ws + (int64_t)hy->n_dec * M * hy->n_splits * D;
      da.out = inst->ao + (int64_t)hy->Tc * M * D;
      da.scale_log2 = a.scale_log2;
      da.order = hy->d_order;
      da.kvmap = inst->attn_tc ? &inst->attn_kvmap : nullptr;
      da.layer = l;
      da.n_layers = inst->L;
      LAUNCH(P_ATTN_DECODE, hy->kv_bytes, hy->n_splits > 1 ? 2 : 1, attn_decode_launch(da, D, st));
    }
    if (inst->tp_fused) {  // O-proj pushing its tiles to the peer, then all-reduce + residual + RMSNorm (N2)
      const int ep = ++inst->tp_epoch;
      GemmEpi eo = tp_push_epi(inst, ep);
      eo.mode = EPI_F32;
      LAUNCH(P_GEMM_PREFILL, 2.0 * T * H * M * D, 1,
             prefill_gemm(inst, inst->m_ao.a, w.o_a, w.o_b, T, H, M * D, eo));
      LAUNCH(P_OTHER, 0, 1, tp_allreduce(inst, ep, T, w.ffn_norm, inst->h));
    } else {
      GemmEpi eo = resid_epi(inst);
      eo.mode = resid_mode_prefill(inst);
      if (dnorm) nrm_out(eo, w.ffn_norm);
      LAUNCH(P_GEMM_PREFILL, 2.0 * T * H * M * D, 1,
             prefill_gemm(inst, inst->m_ao.a, w.o_a, w.o_b, T, H, M * D, eo));
      ALLREDUCE_X(T);
      if (dnorm) ss_ready = true;
      else LAUNCH(P_OTHER, 0, 1, rmsnorm_launch(inst->x, H, nullptr, w.ffn_norm, inst->h, T, H, eps, st));
    }
    GemmEpi eg = epi_base(inst);
    nrm_in(eg);
    ss_ready = false;
    eg.mode = EPI_SILU;
    eg.out = inst->act;
    eg.ldo = F;
    LAUNCH(P_GEMM_PREFILL, 2.0 * T * 2 * F * H, 1,
           prefill_gemm(inst, inst->m_h.a, w.gu_a, w.gu_b, T, 2 * F, H, eg));
    if (inst->tp_fused) {  // the next layer's attention norm rides along (the final norm is the LM head's)
      const int ep = ++inst->tp_epoch;
      GemmEpi ed = tp_push_epi(inst, ep);
      ed.mode = EPI_F32;
      LAUNCH(P_GEMM_PREFILL, 2.0 * T * H * F, 1,
             prefill_gemm(inst, inst->m_act.a, w.d_a, w.d_b, T, H, F, ed));
      const bool last = l + 1 == L;
      LAUNCH(P_OTHER, 0, 1, tp_allreduce(inst, ep, T, last ? nullptr : inst->lw[l + 1].attn_norm, inst->h));
      h_ready = !last;
    } else {
      GemmEpi ed = resid_epi(inst);
      ed.mode = resid_mode_prefill(inst);
      const bool last = l + 1 == L;  // (the LM head normalises its rows itself)
      if (dnorm && !last) nrm_out(ed, inst->lw[l + 1].attn_norm);
      LAUNCH(P_GEMM_PREFILL, 2.0 * T * H * F, 1,
             prefill_gemm(inst, inst->m_act.a, w.d_a, w.d_b, T, H, F, ed));
      ALLREDUCE_X(T);
      if (dnorm && !last) h_ready = ss_ready = true;
    }
    if (inst->debug)
      CK(cudaMemcpyAsync(inst->dbg + (int64_t)(l + 1) * inst->T_max * H, inst->x, sizeof(float) * (int64_t)T * H,
                         cudaMemcpyDeviceToDevice, st));
  }
  return ECOSERVE_OK;
}

// d_skp / sk_grid / sk_maxp: the stream-K decode attention (attention.cu) when sk_grid > 0
struct SkAttn {
  const int* d_skp = nullptr;  // [B + 1] block prefix over the LPT ranks
  int grid = 0, maxp = 0;
};

static void set_sk(ecoserve_instance* inst, DecodeAttnArgs& a, const SkAttn& sk) {
  if (sk.grid <= 0) return;
  a.sk_prefix = sk.d_skp;
  a.sk_cnt = inst->sk_cnt;
  a.sk_grid = sk.grid;
  a.sk_maxp = sk.maxp;
  a.n_splits = 1;
}

static ecoserve_status run_layers_decode(ecoserve_instance* inst, int B, const int* d_ids, const int* d_pos,
                                         const int* d_slot, const int* d_ctx, const int* d_bt, int bt_ld,
                                         int max_blocks, double kv_bytes, bool* final_normed,
                                         const int* d_order = nullptr, SkAttn sk = SkAttn()) {
  cudaStream_t st = inst->stream;
  const int L = inst->L, H = inst->H, M = inst->M, D = inst->D, F = inst->F;
  const float eps = inst->shape.rms_eps;
  LAUNCH(P_OTHER, 0, 1, embed_launch(d_ids, inst->embed, inst->x, B, H, inst->V, st));
  if (inst->debug) CK(cudaMemcpyAsync(inst->dbg, inst->x, sizeof(float) * (int64_t)B * H, cudaMemcpyDeviceToDevice, st));
  int bps = 1;
  int n_splits = decode_attn_splits(inst, B, max_blocks, &bps);
  if ((int64_t)B * M * n_splits * (D + 2) > inst->attn_ws_elems) return ECOSERVE_ERR_INVALID_ARG;
  // RMSNorms fused into the split-K reduction of the preceding O / down projection (TP=1)
  const bool can_fuse = inst->tp == 1;
  if (inst->chain) {
    // layer 0's attention input: norm + QKV (+ RoPE, KV write) as separate kernels, then per
    // layer the attention and one chain kernel (O ... next layer's QKV, see build_chain)
    LAUNCH(P_OTHER, 0, 1, rmsnorm_launch(inst->x, H, nullptr, inst->lw[0].attn_norm, inst->h, B, H, eps, st));
    {
      GemmEpi e = epi_base(inst);
      e.pos = d_pos;
      e.slot = d_slot;
      e.k_cache = k_layer(inst, 0);
      e.v_cache = v_layer(inst, 0);
      int nk = 0;
      LAUNCH(P_GEMM_DECODE, 2.0 * inst->QKV * H, nk,
             decode_gemm(inst, inst->lw[0].qkv_a, inst->m_h, inst->QKV, H, B, EPI_SWAP_QKV, e, &nk, nullptr, nullptr,
                         nullptr, &inst->lw[0].qkv_b));
    }
    ChainCall cc;
    cc.n_tok = B;
    cc.ss_ld = inst->chain_ss_ld;
    cc.ws = inst->chain_ws;
    cc.pos = d_pos;
    cc.slot = d_slot;
    cc.bar = inst->chain_bar;
    cc.err = inst->chain_err;
    cc.trace = nullptr;
    static const char* trace_path = getenv("ECOSERVE_CHAIN_TRACE");  // debug: marks of layer 1's chain
    if (trace_path && !inst->chain_trace)
      CK(cudaMalloc(&inst->chain_trace, sizeof(unsigned long long) * inst->num_sms * 32 * 4));
    for (int l = 0; l < L; ++l) {
      DecodeAttnArgs a;
      a.q = inst->q;
      a.k_cache = k_layer(inst, l);
      a.v_cache = v_layer(inst, l);
      a.blk_stride = inst->blk_stride;
      a.ctx_lens = d_ctx;
      a.block_tables = d_bt;
      a.bt_ld = bt_ld;
      a.B = B;
      a.n_heads = M;
      a.n_kv = inst->Mkv;
      a.n_splits = n_splits;
      a.blocks_per_split = bps;
      a.part_o = inst->attn_ws;
      a.part_ml = inst->attn_ws + (int64_t)B * M * n_splits * D;
      a.out = inst->ao;
      a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
      a.order = d_order;
      a.kvmap = inst->attn_tc ? &inst->attn_kvmap : nullptr;
      a.layer = l;
      a.n_layers = L;
      set_sk(inst, a, sk);
      LAUNCH(P_ATTN_DECODE, kv_bytes, a.n_splits > 1 ? 2 : 1, attn_decode_launch(a, D, st));
      cc.bar_base = inst->chain_base;
      cc.trace = (trace_path && l == std::min(1, L - 1)) ? inst->chain_trace : nullptr;
      const int n = inst->chain_n[l];
      const double bytes = inst->chain_bytes_layer - (l + 1 == L ? 2.0 * inst->QKV * H : 0.0);
      LAUNCH(P_GEMM_DECODE, bytes, 1,
             decode_chain_launch(inst->d_chain + inst->chain_off[l], n, cc, inst->num_sms, st));
      inst->chain_base += (unsigned long long)n * inst->num_sms;
      if (inst->debug)
        CK(cudaMemcpyAsync(inst->dbg + (int64_t)(l + 1) * inst->T_max * H, inst->x, sizeof(float) * (int64_t)B * H,
                           cudaMemcpyDeviceToDevice, st));
    }
    *final_normed = true;
    if (trace_path) {  // append "cta step k t_ns" lines (relative to the earliest mark)
      std::vector<unsigned long long> t((size_t)inst->num_sms * 32 * 4);
      CK(cudaMemcpyAsync(t.data(), inst->chain_trace, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      unsigned long long t0 = ~0ull;
      for (int c = 0; c < inst->num_sms; ++c) t0 = std::min(t0, t[(size_t)(c * 32) * 4 + 3]);
      FILE* f = fopen(trace_path, "a");
      if (f) {
        fprintf(f, "# B=%d steps=%d\n", B, inst->chain_n[std::min(1, L - 1)]);
        for (int c = 0; c < inst->num_sms; ++c)
          for (int si = 0; si < inst->chain_n[std::min(1, L - 1)]; ++si)
            for (int k = 0; k < 4; ++k) {
              const unsigned long long v = t[((size_t)c * 32 + si) * 4 + k];
              if (v >= t0 && v - t0 < 1000000000ull) fprintf(f, "%d %d %d %llu\n", c, si, k, v - t0);
            }
        fclose(f);
      }
      CK(cudaMemsetAsync(inst->chain_trace, 0, sizeof(unsigned long long) * t.size(), st));
    }
    return ECOSERVE_OK;
  }
  if (use_flow(inst, B)) {
    // per layer: QKV GEMM (+ split reduction with RoPE / KV write, scaled by the 1/rms the
    // previous flow kernel left in flow_rvec) -> attention -> one flow kernel (O, gate/up,
    // down; decode_flow.cu) that leaves x, h = bf16(x * next gamma) and flow_rvec
    LAUNCH(P_OTHER, 0, 1, rmsnorm_launch(inst->x, H, nullptr, inst->lw[0].attn_norm, inst->h, B, H, eps, st));
    const int bn = B <= 64 ? 64 : 128;
    const int bi = bn_index(bn);
    const double flow_bytes = 2.0 * ((double)H * M * D + 2.0 * F * H + (double)H * F);
    const int nt_o = H / 128;
    for (int l = 0; l < L; ++l) {
      LayerW& w = inst->lw[l];
      GemmEpi e = epi_base(inst);
      e.pos = d_pos;
      e.slot = d_slot;
      e.k_cache = k_layer(inst, l);
      e.v_cache = v_layer(inst, l);
      if (l > 0) e.rvec = inst->flow_rvec;
      int nk = 0;
      LAUNCH(P_GEMM_DECODE, 2.0 * inst->QKV * H, nk,
             decode_gemm(inst, w.qkv_a, inst->m_h, inst->QKV, H, B, EPI_SWAP_QKV, e, &nk, nullptr, nullptr, nullptr,
                         &w.qkv_b));
      DecodeAttnArgs a;
      a.q = inst->q;
      a.k_cache = k_layer(inst, l);
      a.v_cache = v_layer(inst, l);
      a.blk_stride = inst->blk_stride;
      a.ctx_lens = d_ctx;
      a.block_tables = d_bt;
      a.bt_ld = bt_ld;
      a.B = B;
      a.n_heads = M;
      a.n_kv = inst->Mkv;
      a.n_splits = n_splits;
      a.blocks_per_split = bps;
      a.part_o = inst->attn_ws;
      a.part_ml = inst->attn_ws + (int64_t)B * M * n_splits * D;
      a.out = inst->ao;
      a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
      a.order = d_order;
      a.kvmap = inst->attn_tc ? &inst->attn_kvmap : nullptr;
      a.layer = l;
      a.n_layers = L;
      set_sk(inst, a, sk);
      LAUNCH(P_ATTN_DECODE, kv_bytes, a.n_splits > 1 ? 2 : 1, attn_decode_launch(a, D, st));
      const bool last = l + 1 == L;
      FlowArgs fa;
      fa.B = B;
      fa.H = H;
      fa.F = F;
      fa.MD = M * D;
      fa.epoch = ++inst->flow_epoch;
      fa.eps = eps;
      fa.inv_h = 1.f / (float)H;
      fa.x = inst->x;
      fa.h = inst->h;
      fa.h_out = last ? inst->hl : inst->h;
      fa.act = inst->act;
      fa.gamma_o = w.ffn_norm;
      fa.gamma_d = last ? inst->final_norm : inst->lw[l + 1].attn_norm;
      fa.ss_o = inst->flow_ss;
      fa.ss_d = inst->flow_ss + nt_o * 128;
      fa.rvec = inst->flow_rvec;
      fa.flags_o = inst->flow_flags;
      fa.flags_gu = inst->flow_flags + flow_gu_flag_off(H);
      fa.cnt = inst->flow_cnt;
      fa.cnt_ld = inst->flow_cnt_ld;
      fa.done_d = inst->flow_cnt + 6 * inst->flow_cnt_ld;
      fa.slots = inst->flow_slots;
      fa.err = inst->flow_err;
      fa.trace = (flow_trace_path() && l == std::min(5, L - 1)) ? inst->flow_trace : nullptr;
      LAUNCH(P_GEMM_DECODE, flow_bytes, 1,
             decode_flow_launch(&w.o_a, &w.gu_a, &w.d_a, &inst->m_ao.b[bi], &inst->m_h.b[bi], &inst->m_act.b[bi],
                                &inst->flow_xmap, &inst->flow_actmap, fa, bn, inst->num_sms, st));
      if (inst->debug)
        CK(cudaMemcpyAsync(inst->dbg + (int64_t)(l + 1) * inst->T_max * H, inst->x, sizeof(float) * (int64_t)B * H,
                           cudaMemcpyDeviceToDevice, st));
    }
    *final_normed = true;  // hl = bf16(x * final_norm): the LM-head argmax is invariant to 1/rms > 0
    if (flow_trace_path()) {  // debug: append "cta mark t_ns" of layer 5's flow kernel
      std::vector<unsigned long long> t((size_t)inst->num_sms * 16);
      CK(cudaMemcpyAsync(t.data(), inst->flow_trace, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      unsigned long long t0 = ~0ull;
      for (int c = 0; c < inst->num_sms; ++c) if (t[c * 16]) t0 = std::min(t0, t[c * 16]);
      FILE* f = fopen(flow_trace_path(), "a");
      if (f) {
        fprintf(f, "# B=%d\n", B);
        for (int c = 0; c < inst->num_sms; ++c)
          for (int k = 0; k < 16; ++k)
            if (t[c * 16 + k] >= t0) fprintf(f, "%d %d %llu\n", c, k, t[c * 16 + k] - t0);
        fclose(f);
      }
      CK(cudaMemsetAsync(inst->flow_trace, 0, sizeof(unsigned long long) * t.size(), st));
    }
    return ECOSERVE_OK;
  }
  bool h_ready = false, fused = false;
  *final_normed = false;
  for (int l = 0; l < L; ++l) {
    LayerW& w = inst->lw[l];
    if (!h_ready) LAUNCH(P_OTHER, 0, 1, rmsnorm_launch(inst->x, H, nullptr, w.attn_norm, inst->h, B, H, eps, st));
    h_ready = false;
    GemmEpi e = epi_base(inst);
    e.pos = d_pos;
    e.slot = d_slot;
    e.k_cache = k_layer(inst, l);
    e.v_cache = v_layer(inst, l);
    int nk = 0;
    const int abl = ablate_mask();
    // QKV split partials reduced (+ RoPE, K/V append) inside the attention kernel (TMA path)
    const bool fuse_qkv = qkv_fuse_enabled() && inst->attn_tc && D == 128;
    int qkv_sp = 0;
    if (!(abl & 4)) {
      if (fuse_qkv)
        LAUNCH(P_GEMM_DECODE, 2.0 * inst->QKV * H, 1,
               decode_partials(inst, w.qkv_a, inst->m_h, inst->QKV, H, B, &qkv_sp));
      else
        LAUNCH(P_GEMM_DECODE, 2.0 * inst->QKV * H, nk,
               decode_gemm(inst, w.qkv_a, inst->m_h, inst->QKV, H, B, EPI_SWAP_QKV, e, &nk, nullptr, nullptr, nullptr,
                           &w.qkv_b));
    }
    DecodeAttnArgs a;
    if (fuse_qkv && qkv_sp > 0) {
      a.qkv_part = inst->part;
      a.qkv_splits = qkv_sp;
      a.qkv_ld = inst->QKV;
      a.pos = d_pos;
      a.slot = d_slot;
      a.rope_cos = inst->rope_cos;
      a.rope_sin = inst->rope_sin;
    }
    a.q = inst->q;
    a.k_cache = k_layer(inst, l);
    a.v_cache = v_layer(inst, l);
    a.blk_stride = inst->blk_stride;
    a.ctx_lens = d_ctx;
    a.block_tables = d_bt;
    a.bt_ld = bt_ld;
    a.B = B;
    a.n_heads = M;
    a.n_kv = inst->Mkv;
    a.n_splits = n_splits;
    a.blocks_per_split = bps;
    a.part_o = inst->attn_ws;
    a.part_ml = inst->attn_ws + (int64_t)B * M * n_splits * D;
    a.out = inst->ao;
    a.scale_log2 = (float)(1.4426950408889634 / sqrt((double)D));
    a.order = d_order;
    a.kvmap = inst->attn_tc ? &inst->attn_kvmap : nullptr;  // TMA staging of K / V (head_dim 128)
    a.layer = l;
    a.n_layers = L;
    set_sk(inst, a, sk);
    if (!(abl & 1)) LAUNCH(P_ATTN_DECODE, kv_bytes, a.n_splits > 1 ? 2 : 1, attn_decode_launch(a, D, st));
    if (abl & 2) {
      h_ready = true;
      continue;
    }
    if (inst->tp_fused) {  // partials -> fused push + all-reduce + residual + RMSNorm over NVLink (N2)
      const int ep = ++inst->tp_epoch;
      int sp = 1;
      if (tp_decode_push_enabled() && 4 * B <= inst->tp_rows_max) {  // [splits <= 4][B][H] fits a plane
        LAUNCH(P_GEMM_DECODE, 2.0 * H * M * D, 1,
               decode_partials_push(inst, w.o_a, inst->m_ao, H, M * D, B, ep, &sp));
        LAUNCH(P_OTHER, 0, 1, tp_allreduce(inst, ep, B, w.ffn_norm, inst->h, sp));
      } else {
        int skp[2] = {0, 0};
        LAUNCH(P_GEMM_DECODE, 2.0 * H * M * D, 1, decode_partials(inst, w.o_a, inst->m_ao, H, M * D, B, &sp, skp));
        LAUNCH(P_OTHER, 0, 1, tp_push_rows(inst, ep, sp, B, w.ffn_norm, inst->h, skp));
      }
    } else {
      GemmEpi eo = resid_epi(inst);
      set_prefetch(inst, eo, 4 * l + 2, 2 * F, H, B);  // gate/up next
      LAUNCH(P_GEMM_DECODE, 2.0 * H * M * D, nk,
             decode_gemm(inst, w.o_a, inst->m_ao, H, M * D, B, resid_mode_decode(inst), eo, &nk,
                         can_fuse ? w.ffn_norm : nullptr, inst->h, &fused, &w.o_b));
      ALLREDUCE_X(B);
      if (!fused) LAUNCH(P_OTHER, 0, 1, rmsnorm_launch(inst->x, H, nullptr, w.ffn_norm, inst->h, B, H, eps, st));
    }
    GemmEpi eg = epi_base(inst);
    eg.out = inst->act;
    eg.ldo = F;
    set_prefetch(inst, eg, 4 * l + 3, H, F, B);  // down next
    inst->gu_trace_layer = l;
    // the down projection's reduction also applies the next RMSNorm: the next layer's
    // attention norm, or after the last layer the final norm (into the LM-head input)
    const bool last = l + 1 == L;
    if (inst->gw_w1 > 0 && B <= 128 && !inst->tp_fused && inst->tp == 1 && decode_variant() == 1) {
      // gate/up in two waves. Its 2F/128 tiles exceed the SMs: in one kernel the second
      // wave leaves the SMs done after one tile waiting (the down GEMM behind it can only
      // prefetch weights). Here wave 1 (W1 = num_sms tiles) runs alone; then the down
      // projection's K blocks [0, W1) -- which read only wave-1 output -- run beside wave 2
      // on the other SMs (wave 2 waits on a flag instead of the kernel before it, see
      // GemmEpi::flag_wait); then the down K blocks [W1, F/64); one reduction sums all
      // split planes in order and applies the next RMSNorm.
      const int W1 = inst->gw_w1, W2 = 2 * F / 128 - W1, dt = H / 128;
      const int bn = B <= 64 ? 64 : 128, bi = bn_index(bn);
      const int s1 = gemm_effective_splits(64 * W1, std::max(1, std::min(4, (inst->num_sms - W2) / dt)));
      const int s2 = gemm_effective_splits(F - 64 * W1, std::max(1, std::min(4, inst->num_sms / dt)));
      const int ep = ++inst->gw_epoch;
      static const char* gw_trace = getenv("ECOSERVE_GW_TRACE");  // debug: per-CTA marks of layer 5
      unsigned long long* tr = nullptr;
      if (gw_trace && l == 5) {
        if (!inst->gw_trace) {
          CK(cudaMalloc(&inst->gw_trace, sizeof(unsigned long long) * 4 * inst->num_sms * 16));
        }
        CK(cudaMemsetAsync(inst->gw_trace, 0, sizeof(unsigned long long) * 4 * inst->num_sms * 16, st));
        tr = inst->gw_trace;
      }
      GemmEpi g1 = eg;
      g1.trace = tr;
      g1.mode = EPI_SWAP_SILU;
      g1.indep = 1;
      g1.pf_map = nullptr;
      g1.flag_set = inst->gw_flag;
      g1.flag_epoch = ep;
      LAUNCH(P_GEMM_DECODE, 2.0 * 128 * W1 * H, 1,
             gemm_launch_r(&w.gu_a, &inst->m_h.b[bi], 128 * W1, B, H, bn, 1, 1, g1, inst->num_sms, st));
      GemmEpi d1 = epi_base(inst);
      d1.mode = EPI_SWAP_F32;
      d1.out = inst->part;
      d1.ldo = H;
      d1.indep = 1;
      d1.trace = tr ? tr + 1 * inst->num_sms * 16 : nullptr;
      LAUNCH(P_GEMM_DECODE, 2.0 * H * 64 * W1, 1,
             gemm_launch_r(&w.d1_a, &inst->act_k1.b[bi], H, B, 64 * W1, bn, 1, s1, d1, inst->num_sms, st));
      GemmEpi g2 = g1;
      g2.out = inst->act + 64LL * W1;
      g2.flag_set = nullptr;
      g2.flag_wait = inst->gw_flag;
      g2.trace = tr ? tr + 2 * inst->num_sms * 16 : nullptr;
      LAUNCH(P_GEMM_DECODE, 2.0 * 128 * W2 * H, 1,
             gemm_launch_r(&w.gu2_a, &inst->m_h.b[bi], 128 * W2, B, H, bn, 1, 1, g2, inst->num_sms, st));
      GemmEpi d2 = d1;
      d2.out = inst->part + (int64_t)s1 * B * H;
      d2.trace = tr ? tr + 3 * inst->num_sms * 16 : nullptr;
      LAUNCH(P_GEMM_DECODE, 2.0 * H * (F - 64.0 * W1), 1,
             gemm_launch_r(&w.d2_a, &inst->act_k2.b[bi], H, B, F - 64 * W1, bn, 1, s2, d2, inst->num_sms, st));
      LAUNCH(P_OTHER, 0, 1,
             splitk_resid_rmsnorm_launch(inst->part, s1 + s2, B, inst->x, last ? inst->final_norm : inst->lw[l + 1].attn_norm,
                                         last ? inst->hl : inst->h, H, eps, st));
      if (tr) {  // append "kernel cta mark t_ns" (relative to the earliest mark)
        std::vector<unsigned long long> t((size_t)4 * inst->num_sms * 16);
        CK(cudaMemcpyAsync(t.data(), tr, sizeof(unsigned long long) * t.size(), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        unsigned long long t0 = ~0ull;
        for (auto v : t)
          if (v) t0 = std::min(t0, v);
        FILE* f = fopen(gw_trace, "a");
        if (f) {
          fprintf(f, "#\n");
          for (int kk = 0; kk < 4; ++kk)
            for (int c = 0; c < inst->num_sms; ++c)
              for (int m = 0; m < 8; ++m) {
                const unsigned long long v = t[((size_t)kk * inst->num_sms + c) * 16 + m];
                if (v) fprintf(f, "%d %d %d %llu\n", kk, c, m, v - t0);
              }
          fclose(f);
        }
      }
      fused = true;
      h_ready = !last;
      if (last) *final_normed = true;
      if (inst->debug)
        CK(cudaMemcpyAsync(inst->dbg + (int64_t)(l + 1) * inst->T_max * H, inst->x, sizeof(float) * (int64_t)B * H,
                           cudaMemcpyDeviceToDevice, st));
      continue;
    }
    LAUNCH(P_GEMM_DECODE, 2.0 * 2 * F * H, nk,
           decode_gemm(inst, w.gu_a, inst->m_h, 2 * F, H, B, EPI_SWAP_SILU, eg, &nk, nullptr, nullptr, nullptr, &w.gu_b));
    if (inst->tp_fused) {
      const int ep = ++inst->tp_epoch;
      int sp = 1;
      const bf16* g_next = last ? inst->final_norm : inst->lw[l + 1].attn_norm;
      bf16* h_next = last ? inst->hl : inst->h;
      if (tp_decode_push_enabled() && 4 * B <= inst->tp_rows_max) {  // [splits <= 4][B][H] fits a plane
        LAUNCH(P_GEMM_DECODE, 2.0 * H * F, 1, decode_partials_push(inst, w.d_a, inst->m_act, H, F, B, ep, &sp));
        LAUNCH(P_OTHER, 0, 1, tp_allreduce(inst, ep, B, g_next, h_next, sp));
      } else {
        int skp[2] = {0, 0};
        LAUNCH(P_GEMM_DECODE, 2.0 * H * F, 1, decode_partials(inst, w.d_a, inst->m_act, H, F, B, &sp, skp));
        LAUNCH(P_OTHER, 0, 1, tp_push_rows(inst, ep, sp, B, g_next, h_next, skp));
      }
      fused = true;
    } else {
      GemmEpi ed = resid_epi(inst);
      if (!last) set_prefetch(inst, ed, 4 * (l + 1), inst->QKV, H, B);  // next layer's QKV
      LAUNCH(P_GEMM_DECODE, 2.0 * H * F, nk,
             decode_gemm(inst, w.d_a, inst->m_act, H, F, B, resid_mode_decode(inst), ed, &nk,
                         can_fuse ? (last ? inst->final_norm : inst->lw[l + 1].attn_norm) : nullptr,
                         last ? inst->hl : inst->h, &fused, &w.d_b));
      ALLREDUCE_X(B);
    }
    h_ready = fused && !last;
    if (last) *final_normed = fused;
    if (inst->debug)
      CK(cudaMemcpyAsync(inst->dbg + (int64_t)(l + 1) * inst->T_max * H, inst->x, sizeof(float) * (int64_t)B * H,
                         cudaMemcpyDeviceToDevice, st));
  }
  return ECOSERVE_OK;
}

// final RMSNorm of the selected rows + LM head + greedy argmax -> h_tokens[0..n)
static ecoserve_status lm_head_argmax(ecoserve_instance* inst, const int* d_rows, int n, int gemm_cls,
                                      bool normed = false) {
  cudaStream_t st = inst->stream;
  const int H = inst->H;
  if (!normed)  // (decode: usually already fused into the last down projection's reduction)
    LAUNCH(P_OTHER, 0, 1,
           rmsnorm_launch(inst->x, H, d_rows, inst->final_norm, inst->hl, n, H, inst->shape.rms_eps, st));
  GemmEpi e;
  memset(&e, 0, sizeof(e));
  e.mode = EPI_SWAP_ARGMAX;
  e.indep = 1;
  e.am_val = inst->am_val;
  e.am_idx = inst->am_idx;
  e.am_ld = inst->am_ld;
  const int bn = pick_bn(n);
  LAUNCH(gemm_cls, gemm_cls == P_GEMM_DECODE ? 2.0 * inst->V * H : 2.0 * inst->V * H * n, 1,
         gemm_launch(&inst->lm_a, &inst->m_hl.b[bn_index(bn)], inst->V, n, H, bn, 1, e, inst->num_sms, st));
  LAUNCH(P_OTHER, 0, 1,
         argmax_reduce_launch(inst->am_val, inst->am_idx, n, inst->am_ld, inst->am_ld, inst->d_tokens, st));
  return ECOSERVE_OK;
}

// Enqueued with the token copy-back: the TP exchange's timeout flag.
static cudaError_t copy_step_flags(ecoserve_instance* inst) {
  if (!inst->tp_err) return cudaSuccess;
  return cudaMemcpyAsync(inst->h_tp_err, inst->tp_err, sizeof(int), cudaMemcpyDeviceToHost, inst->stream);
}

// After the step synchronised: a TP exchange that timed out (the peer stopped
// mid-phase) and NaN rows, whose argmax is ECO_TOKEN_NAN (reading A6; feeding it back
// would embed a garbage id), both mark the instance dead.
static ecoserve_status check_tokens(ecoserve_instance* inst, int n) {
  if (inst->h_tp_err && *inst->h_tp_err) {
    inst->err = "TP=2 exchange: the peer rank's flag did not arrive within the timeout (peer failed or "
                "stopped mid-phase); instance marked dead";
    inst->dead = true;
    return ECOSERVE_ERR_NCCL;
  }
  for (int i = 0; i < n; ++i)
    if (inst->h_tokens[i] < 0 || inst->h_tokens[i] >= inst->V) {
      inst->err = "NaN logits in LM-head row " + std::to_string(i) + " (reading A6); instance marked dead";
      inst->dead = true;
      return ECOSERVE_ERR_NUMERIC;
    }
  return ECOSERVE_OK;
}

extern "C" {

ecoserve_status ecoserve_prefill_phase(ecoserve_instance* inst, const ecoserve_request* reqs, int32_t n,
                                       int32_t* first_tokens) {
  if (!inst) return ECOSERVE_ERR_INVALID_ARG;
  if (inst->dead) return ECOSERVE_ERR_CUDA;
  if (n < 0 || (n > 0 && (!reqs || !first_tokens))) return ECOSERVE_ERR_INVALID_ARG;
  if (n == 0) return ECOSERVE_OK;
  CK(cudaSetDevice(inst->device));  // the calling thread may have another current device
  // ---- validate everything first (all-or-nothing)
  int64_t need_blocks = 0;
  {
    std::unordered_map<int64_t, int> seen;
    for (int i = 0; i < n; ++i) {
      const ecoserve_request& r = reqs[i];
      if (r.prompt_len < 1 || !r.prompt || r.max_new_tokens < 1 || r.prompt_len > inst->T_max ||
          r.prompt_len + r.max_new_tokens > inst->P_max) {
        inst->err = "invalid request " + std::to_string(r.req_id);
        return ECOSERVE_ERR_INVALID_ARG;
      }
      for (int t = 0; t < r.prompt_len; ++t)
        if (r.prompt[t] < 0 || r.prompt[t] >= inst->V) {
          inst->err = "token id out of range in request " + std::to_string(r.req_id);
          return ECOSERVE_ERR_INVALID_ARG;
        }
      if (inst->reqs.count(r.req_id) || seen.count(r.req_id)) {
        inst->err = "duplicate req_id " + std::to_string(r.req_id);
        return ECOSERVE_ERR_STATE;
      }
      seen[r.req_id] = i;
      need_blocks += (r.prompt_len + BLOCK - 1) / BLOCK;
    }
  }
  if (need_blocks > (int64_t)inst->free_blocks.size()) {
    inst->err = "KV pool exhausted";
    return ECOSERVE_ERR_KV_EXHAUSTED;
  }
  // ---- allocate and register
  std::vector<Req*> rs(n);
  for (int i = 0; i < n; ++i) {
    Req r;
    r.id = reqs[i].req_id;
    r.S = reqs[i].prompt_len;
    r.max_new = reqs[i].max_new_tokens;
    r.prompt.assign(reqs[i].prompt, reqs[i].prompt + r.S);
    r.prefilled = r.S;
    const int nb = (r.S + BLOCK - 1) / BLOCK;
    for (int b = 0; b < nb; ++b) {
      r.blocks.push_back(inst->free_blocks.back());
      inst->free_blocks.pop_back();
    }
    rs[i] = &(inst->reqs[r.id] = std::move(r));
  }
  // ---- batches of <= T_max tokens and <= B_max sequences (FIFO, reading A16)
  inst->dbg_rows.clear();
  int i0 = 0;
  while (i0 < n) {
    int i1 = i0, tok = 0;
    while (i1 < n && (i1 == i0 || (tok + rs[i1]->S <= inst->T_max && i1 - i0 < inst->B_max))) tok += rs[i1++]->S;
    const int ns = i1 - i0;
    int bt_ld = 1;
    for (int i = i0; i < i1; ++i) bt_ld = std::max(bt_ld, (int)rs[i]->blocks.size());
    // q tiles, longest-first
    std::vector<std::pair<int, int>> tiles;
    for (int i = i0; i < i1; ++i)
      for (int qs = 0; qs < rs[i]->S; qs += inst->attn_tc ? 128 : 64) tiles.push_back({i - i0, qs});
    std::stable_sort(tiles.begin(), tiles.end(),
                     [](const std::pair<int, int>& a, const std::pair<int, int>& b) { return a.second > b.second; });
    // pack metadata: ids[T] pos[T] slot[T] cu[ns+1] rows[ns] bt[ns][bt_ld] tiles[2*nt]
    int* hm = inst->h_meta;
    int* ids = hm;
    int* pos = ids + tok;
    int* slot = pos + tok;
    int* cu = slot + tok;
    int* rows = cu + ns + 1;
    int* bt = rows + ns;
    int* tl = bt + ns * bt_ld;
    const int64_t used = (tl - hm) + 2LL * tiles.size();
    if (used > inst->meta_cap) {
      inst->err = "metadata buffer too small";
      return ECOSERVE_ERR_INVALID_ARG;
    }
    int t = 0;
    for (int i = i0; i < i1; ++i) {
      Req* r = rs[i];
      cu[i - i0] = t;
      for (int p = 0; p < r->S; ++p, ++t) {
        ids[t] = r->prompt[p];
        pos[t] = p;
        slot[t] = r->blocks[p / BLOCK] * BLOCK + p % BLOCK;
      }
      rows[i - i0] = t - 1;
      for (int b = 0; b < bt_ld; ++b) bt[(i - i0) * bt_ld + b] = b < (int)r->blocks.size() ? r->blocks[b] : 0;
      if (inst->debug) inst->dbg_rows[r->id] = {cu[i - i0], r->S};
    }
    cu[ns] = t;
    for (size_t k = 0; k < tiles.size(); ++k) {
      tl[2 * k] = tiles[k].first;
      tl[2 * k + 1] = tiles[k].second;
    }
    cudaStream_t st = inst->stream;
    CK(cudaMemcpyAsync(inst->d_meta, hm, sizeof(int) * used, cudaMemcpyHostToDevice, st));
    int* d = inst->d_meta;
    double attn_flop = 0;  // causal QK^T + PV: 2 * 2 * M * D * S(S+1)/2 per sequence
    for (int i = i0; i < i1; ++i) attn_flop += 2.0 * inst->M * inst->D * (double)rs[i]->S * (rs[i]->S + 1);
    const int pm = inst->prof.begin(P_PREFILL, st);
    ecoserve_status s = run_layers_prefill(inst, tok, d, d + (pos - hm), d + (slot - hm), d + (cu - hm),
                                           d + (bt - hm), bt_ld, d + (tl - hm), (int)tiles.size(), attn_flop);
    if (s != ECOSERVE_OK) return s;
    s = lm_head_argmax(inst, d + (rows - hm), ns, P_OTHER);
    if (s != ECOSERVE_OK) return s;
    inst->prof.end(pm, tok, st);
    CK(cudaMemcpyAsync(inst->h_tokens, inst->d_tokens, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
    CK(copy_step_flags(inst));
    CK(cudaStreamSynchronize(st));
    inst->prof.resolve();
    inst->prof.tokens[0] += tok;
    inst->prof.h2d += sizeof(int) * used;
    inst->prof.d2h += sizeof(int) * ns;
    if (ecoserve_status ts = check_tokens(inst, ns); ts != ECOSERVE_OK) return ts;
    for (int i = i0; i < i1; ++i) {
      Req* r = rs[i];
      r->last_token = inst->h_tokens[i - i0];
      r->n_gen = 1;
      r->finished = r->n_gen >= r->max_new;
      first_tokens[i] = r->last_token;
    }
    i0 = i1;
  }
  return ECOSERVE_OK;
}

// ---------------------------------------------------------------- hybrid batches (N3)
ecoserve_status ecoserve_hybrid_step(ecoserve_instance* inst, const ecoserve_chunk* chunks, int32_t n_chunks,
                                     const int64_t* decode_ids, int32_t n_decode, int32_t* chunk_tokens,
                                     int32_t* decode_tokens) {
  if (!inst) return ECOSERVE_ERR_INVALID_ARG;
  if (inst->dead) return ECOSERVE_ERR_CUDA;
  if (n_chunks < 0 || n_decode < 0 || (n_chunks > 0 && (!chunks || !chunk_tokens)) ||
      (n_decode > 0 && (!decode_ids || !decode_tokens)) || n_chunks + n_decode > inst->B_max)
    return ECOSERVE_ERR_INVALID_ARG;
  if (n_chunks + n_decode == 0) return ECOSERVE_OK;
  CK(cudaSetDevice(inst->device));
  // ---- validate (all-or-nothing)
  int Tc = 0;
  int64_t need = 0;
  std::unordered_map<int64_t, int> seen;
  for (int i = 0; i < n_chunks; ++i) {
    const ecoserve_chunk& c = chunks[i];
    if (c.chunk_len < 1 || seen.count(c.req_id)) return ECOSERVE_ERR_INVALID_ARG;
    seen[c.req_id] = i;
    auto it = inst->reqs.find(c.req_id);
    int pre = 0, S = 0, have = 0;
    if (it == inst->reqs.end()) {  // first chunk of a new request
      if (!c.prompt || c.prompt_len < 1 || c.max_new_tokens < 1 || c.prompt_len + c.max_new_tokens > inst->P_max) {
        inst->err = "invalid request " + std::to_string(c.req_id);
        return ECOSERVE_ERR_INVALID_ARG;
      }
      for (int t = 0; t < c.prompt_len; ++t)
        if (c.prompt[t] < 0 || c.prompt[t] >= inst->V) {
          inst->err = "token id out of range in request " + std::to_string(c.req_id);
          return ECOSERVE_ERR_INVALID_ARG;
        }
      S = c.prompt_len;
    } else {
      if (it->second.n_gen > 0) {
        inst->err = "chunk for an already prefilled request " + std::to_string(c.req_id);
        return ECOSERVE_ERR_STATE;
      }
      pre = it->second.prefilled;
      S = it->second.S;
      have = (int)it->second.blocks.size();
    }
    if (pre + c.chunk_len > S) return ECOSERVE_ERR_INVALID_ARG;
    need += std::max(0, (pre + c.chunk_len + BLOCK - 1) / BLOCK - have);
    Tc += c.chunk_len;
  }
  std::vector<Req*> ds(n_decode);
  for (int k = 0; k < n_decode; ++k) {
    auto it = inst->reqs.find(decode_ids[k]);
    if (it == inst->reqs.end() || it->second.n_gen < 1 || it->second.finished || seen.count(decode_ids[k])) {
      inst->err = "hybrid decode of an unknown, unprefilled, finished or chunked req_id " +
                  std::to_string(decode_ids[k]);
      return ECOSERVE_ERR_STATE;
    }
    seen[decode_ids[k]] = -1 - k;
    ds[k] = &it->second;
    const int p = ds[k]->S + ds[k]->n_gen - 1;
    if (p / BLOCK >= (int)ds[k]->blocks.size()) ++need;
  }
  const int T = Tc + n_decode;
  if (T > inst->T_max) return ECOSERVE_ERR_INVALID_ARG;
  if (need > (int64_t)inst->free_blocks.size()) {
    inst->err = "KV pool exhausted";
    return ECOSERVE_ERR_KV_EXHAUSTED;
  }
  // ---- register new requests, allocate blocks
  std::vector<Req*> cs(n_chunks);
  std::vector<int> pre(n_chunks);
  for (int i = 0; i < n_chunks; ++i) {
    const ecoserve_chunk& c = chunks[i];
    auto it = inst->reqs.find(c.req_id);
    if (it == inst->reqs.end()) {
      Req r;
      r.id = c.req_id;
      r.S = c.prompt_len;
      r.max_new = c.max_new_tokens;
      r.prompt.assign(c.prompt, c.prompt + r.S);
      it = inst->reqs.emplace(r.id, std::move(r)).first;
    }
    cs[i] = &it->second;
    pre[i] = cs[i]->prefilled;
    while ((int)cs[i]->blocks.size() * BLOCK < pre[i] + c.chunk_len) {
      cs[i]->blocks.push_back(inst->free_blocks.back());
      inst->free_blocks.pop_back();
    }
  }
  for (int k = 0; k < n_decode; ++k) {
    const int p = ds[k]->S + ds[k]->n_gen - 1;
    if (p / BLOCK >= (int)ds[k]->blocks.size()) {
      ds[k]->blocks.push_back(inst->free_blocks.back());
      inst->free_blocks.pop_back();
    }
  }
  // ---- metadata: ids pos slot [T] | cu [nc+1] | off [nc] | bt_c [nc][ld] | tiles | ctx [nd] | bt_d [nd][ld] | ord [nd] | lm rows
  int bt_ld = 1, max_blocks = 1;
  for (Req* r : cs) bt_ld = std::max(bt_ld, (int)r->blocks.size());
  for (Req* r : ds) {
    bt_ld = std::max(bt_ld, (int)r->blocks.size());
    max_blocks = std::max(max_blocks, (int)r->blocks.size());
  }
  const int qt = inst->attn_tc ? 128 : 64;
  std::vector<std::pair<int, int>> tiles;
  for (int i = 0; i < n_chunks; ++i)
    for (int qs = 0; qs < chunks[i].chunk_len; qs += qt) tiles.push_back({i, qs});
  std::stable_sort(tiles.begin(), tiles.end(), [&](const std::pair<int, int>& a, const std::pair<int, int>& b) {
    return pre[a.first] + a.second > pre[b.first] + b.second;  // most keys first
  });
  int* hm = inst->h_meta;
  int* ids = hm;
  int* pos = ids + T;
  int* slot = pos + T;
  int* cu = slot + T;
  int* off = cu + n_chunks + 1;
  int* bt_c = off + n_chunks;
  int* tl = bt_c + (int64_t)n_chunks * bt_ld;
  int* ctx = tl + 2 * tiles.size();
  int* bt_d = ctx + n_decode;
  int* ord = bt_d + (int64_t)n_decode * bt_ld;
  int* lm = ord + n_decode;
  const int64_t used = (lm - hm) + n_chunks + n_decode;
  if (used > inst->meta_cap) {
    inst->err = "metadata buffer too small";
    return ECOSERVE_ERR_INVALID_ARG;
  }
  int t = 0, nl = 0;
  double attn_flop = 0;
  std::vector<int> completes(n_chunks, 0);
  for (int i = 0; i < n_chunks; ++i) {
    Req* r = cs[i];
    const int len = chunks[i].chunk_len;
    cu[i] = t;
    off[i] = pre[i];
    for (int j = 0; j < len; ++j, ++t) {
      const int p = pre[i] + j;
      ids[t] = r->prompt[p];
      pos[t] = p;
      slot[t] = r->blocks[p / BLOCK] * BLOCK + p % BLOCK;
    }
    for (int b = 0; b < bt_ld; ++b) bt_c[(int64_t)i * bt_ld + b] = b < (int)r->blocks.size() ? r->blocks[b] : 0;
    attn_flop += 4.0 * inst->M * inst->D * ((double)len * pre[i] + 0.5 * len * (len + 1.0));
    if (pre[i] + len == r->S) {
      completes[i] = 1;
      lm[nl++] = t - 1;
    }
  }
  cu[n_chunks] = t;
  for (size_t k = 0; k < tiles.size(); ++k) {
    tl[2 * k] = tiles[k].first;
    tl[2 * k + 1] = tiles[k].second;
  }
  double kv_tokens = 0;
  for (int k = 0; k < n_decode; ++k, ++t) {
    Req* r = ds[k];
    const int p = r->S + r->n_gen - 1;
    ids[t] = r->last_token;
    pos[t] = p;
    slot[t] = r->blocks[p / BLOCK] * BLOCK + p % BLOCK;
    ctx[k] = p + 1;
    kv_tokens += p + 1;
    for (int b = 0; b < bt_ld; ++b) bt_d[(int64_t)k * bt_ld + b] = b < (int)r->blocks.size() ? r->blocks[b] : 0;
    lm[nl++] = t;
  }
  for (int k = 0; k < n_decode; ++k) ord[k] = k;
  std::stable_sort(ord, ord + n_decode, [ctx](int x, int y) { return ctx[x] > ctx[y]; });
  HybridTail hy;
  int* d = inst->d_meta;
  hy.Tc = Tc;
  hy.d_ctx_off = d + (off - hm);
  hy.n_dec = n_decode;
  hy.d_ctx = d + (ctx - hm);
  hy.d_bt = d + (bt_d - hm);
  hy.bt_ld = bt_ld;
  hy.d_order = d + (ord - hm);
  if (n_decode > 0) {
    hy.n_splits = decode_attn_splits(inst, n_decode, max_blocks, &hy.bps);
    if ((int64_t)n_decode * inst->M * hy.n_splits * (inst->D + 2) > inst->attn_ws_elems) return ECOSERVE_ERR_INVALID_ARG;
  }
  hy.kv_bytes = kv_tokens * 2.0 * inst->Mkv * inst->D * 2.0;
  cudaStream_t st = inst->stream;
  CK(cudaMemcpyAsync(inst->d_meta, hm, sizeof(int) * used, cudaMemcpyHostToDevice, st));
  const int pm = inst->prof.begin(Tc > 0 ? P_PREFILL : P_DECODE, st);
  inst->dbg_rows.clear();
  for (int i = 0; i < n_chunks; ++i)
    if (inst->debug) inst->dbg_rows[cs[i]->id] = {cu[i], chunks[i].chunk_len};
  for (int k = 0; k < n_decode; ++k)
    if (inst->debug) inst->dbg_rows[ds[k]->id] = {Tc + k, 1};
  ecoserve_status es = run_layers_prefill(inst, T, d, d + (pos - hm), d + (slot - hm), d + (cu - hm), d + (bt_c - hm),
                                          bt_ld, d + (tl - hm), (int)tiles.size(), attn_flop, &hy);
  if (es != ECOSERVE_OK) return es;
  if (nl > 0) {
    es = lm_head_argmax(inst, d + (lm - hm), nl, P_OTHER);
    if (es != ECOSERVE_OK) return es;
  }
  inst->prof.end(pm, T, st);
  if (nl > 0) CK(cudaMemcpyAsync(inst->h_tokens, inst->d_tokens, sizeof(int) * nl, cudaMemcpyDeviceToHost, st));
  CK(copy_step_flags(inst));
  CK(cudaStreamSynchronize(st));
  inst->prof.resolve();
  inst->prof.tokens[0] += Tc;
  inst->prof.tokens[1] += n_decode;
  inst->prof.h2d += sizeof(int) * used;
  inst->prof.d2h += sizeof(int) * nl;
  if (ecoserve_status ts = check_tokens(inst, nl); ts != ECOSERVE_OK) return ts;
  int li = 0;
  for (int i = 0; i < n_chunks; ++i) {
    Req* r = cs[i];
    r->prefilled = pre[i] + chunks[i].chunk_len;
    chunk_tokens[i] = -1;
    if (completes[i]) {
      r->last_token = inst->h_tokens[li++];
      r->n_gen = 1;
      r->finished = r->n_gen >= r->max_new;
      chunk_tokens[i] = r->last_token;
    }
  }
  for (int k = 0; k < n_decode; ++k) {
    Req* r = ds[k];
    r->last_token = inst->h_tokens[li++];
    r->n_gen += 1;
    r->finished = r->n_gen >= r->max_new;
    decode_tokens[k] = r->last_token;
  }
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_decode_phase(ecoserve_instance* inst, const int64_t* req_ids, int32_t n, int32_t steps,
                                      int32_t* tokens, int32_t* n_finished) {
  if (!inst) return ECOSERVE_ERR_INVALID_ARG;
  if (inst->dead) return ECOSERVE_ERR_CUDA;
  if (n < 0 || steps < 0 || (n > 0 && (!req_ids || !tokens))) return ECOSERVE_ERR_INVALID_ARG;
  if (n > inst->B_max) return ECOSERVE_ERR_INVALID_ARG;
  CK(cudaSetDevice(inst->device));
  std::vector<Req*> rs(n);
  std::unordered_map<int64_t, int> seen;
  for (int i = 0; i < n; ++i) {
    if (seen.count(req_ids[i])) {  // two rows of one request would share a KV slot
      inst->err = "duplicate req_id " + std::to_string(req_ids[i]) + " in the decode set";
      return ECOSERVE_ERR_INVALID_ARG;
    }
    seen[req_ids[i]] = i;
    auto it = inst->reqs.find(req_ids[i]);
    if (it == inst->reqs.end() || it->second.n_gen < 1) {
      inst->err = "decode of unknown or unprefilled req_id " + std::to_string(req_ids[i]);
      return ECOSERVE_ERR_STATE;
    }
    rs[i] = &it->second;
  }
  for (int i = 0; i < n * steps; ++i) tokens[i] = -1;
  for (int s = 0; s < steps; ++s) {
    std::vector<int> live;
    for (int i = 0; i < n; ++i)
      if (!rs[i]->finished) live.push_back(i);
    const int B = (int)live.size();
    if (B == 0) break;
    // blocks for the token fed at position S + n_gen - 1
    int need = 0;
    for (int i : live) {
      const int p = rs[i]->S + rs[i]->n_gen - 1;
      if (p / BLOCK >= (int)rs[i]->blocks.size()) ++need;
    }
    if (need > (int)inst->free_blocks.size()) {
      inst->err = "KV pool exhausted during decode";
      return ECOSERVE_ERR_KV_EXHAUSTED;
    }
    int bt_ld = 1, max_blocks = 1;
    for (int i : live) {
      Req* r = rs[i];
      const int p = r->S + r->n_gen - 1;
      if (p / BLOCK >= (int)r->blocks.size()) {
        r->blocks.push_back(inst->free_blocks.back());
        inst->free_blocks.pop_back();
      }
      bt_ld = std::max(bt_ld, (int)r->blocks.size());
    }
    max_blocks = bt_ld;
    int* hm = inst->h_meta;
    int* ids = hm;
    int* pos = ids + B;
    int* slot = pos + B;
    int* ctx = slot + B;
    int* rows = ctx + B;
    int* bt = rows + B;
    int* ord = bt + (int64_t)B * bt_ld;  // decode attention: longest context first
    int* skp = ord + B;                  // [B + 1] stream-K attention: block prefix over LPT ranks
    const int64_t used = (skp - hm) + B + 1;
    if (used > inst->meta_cap) return ECOSERVE_ERR_INVALID_ARG;
    if (inst->debug) inst->dbg_rows.clear();
    for (int k = 0; k < B; ++k) {
      Req* r = rs[live[k]];
      const int p = r->S + r->n_gen - 1;
      ids[k] = r->last_token;
      pos[k] = p;
      slot[k] = r->blocks[p / BLOCK] * BLOCK + p % BLOCK;
      ctx[k] = p + 1;
      rows[k] = k;
      for (int b = 0; b < bt_ld; ++b) bt[k * bt_ld + b] = b < (int)r->blocks.size() ? r->blocks[b] : 0;
      if (inst->debug) inst->dbg_rows[r->id] = {k, 1};
    }
    for (int k = 0; k < B; ++k) ord[k] = k;
    std::stable_sort(ord, ord + B, [ctx](int x, int y) { return ctx[x] > ctx[y]; });
    SkAttn sk;
    {
      int max_nb = 0, min_nb = 1 << 30;
      skp[0] = 0;
      for (int r = 0; r < B; ++r) {
        const int nb = (ctx[ord[r]] + 63) / 64;
        skp[r + 1] = skp[r] + nb;
        max_nb = std::max(max_nb, nb);
        min_nb = std::min(min_nb, nb);
      }
      if (inst->attn_tc)
        sk.grid = attn_decode_sk_grid(skp[B] * inst->Mkv, max_nb, min_nb, inst->M, inst->Mkv, inst->D, inst->num_sms,
                                      &sk.maxp);
    }
    cudaStream_t st = inst->stream;
    CK(cudaMemcpyAsync(inst->d_meta, hm, sizeof(int) * used, cudaMemcpyHostToDevice, st));
    int* d = inst->d_meta;
    sk.d_skp = d + (skp - hm);
    double kv_tokens = 0;
    for (int k = 0; k < B; ++k) kv_tokens += ctx[k];
    const double kv_bytes = kv_tokens * 2.0 * inst->Mkv * inst->D * 2.0;  // K and V, one layer
    const int pm = inst->prof.begin(P_DECODE, st);
    const auto t_enq0 = std::chrono::steady_clock::now();
    bool final_normed = false;
    ecoserve_status es = run_layers_decode(inst, B, d, d + (pos - hm), d + (slot - hm), d + (ctx - hm), d + (bt - hm),
                                           bt_ld, max_blocks, kv_bytes, &final_normed, d + (ord - hm), sk);
    if (es != ECOSERVE_OK) return es;
    es = lm_head_argmax(inst, d + (rows - hm), B, P_GEMM_DECODE, final_normed);
    if (es != ECOSERVE_OK) return es;
    inst->prof.end(pm, B, st);
    CK(cudaMemcpyAsync(inst->h_tokens, inst->d_tokens, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
    if (inst->chain) CK(cudaMemcpyAsync(inst->h_chain_err, inst->chain_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (inst->flow) CK(cudaMemcpyAsync(inst->h_flow_err, inst->flow_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (inst->gu_sk) CK(cudaMemcpyAsync(inst->h_gu_err, inst->gu_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(copy_step_flags(inst));
    const auto t_enq1 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(st));
    if (inst->gu_trace && gu_trace_path()) {  // debug: "cta mark t_ns" of layer 5's gate/up launch
      std::vector<unsigned long long> tr((size_t)inst->num_sms * 16);
      CK(cudaMemcpy(tr.data(), inst->gu_trace, sizeof(unsigned long long) * tr.size(), cudaMemcpyDeviceToHost));
      unsigned long long t0 = ~0ull;
      for (int c = 0; c < inst->num_sms; ++c) if (tr[c * 16]) t0 = std::min(t0, tr[c * 16]);
      FILE* f = fopen(gu_trace_path(), "a");
      if (f) {
        fprintf(f, "# B=%d\n", B);
        for (int c = 0; c < inst->num_sms; ++c)
          for (int k = 0; k < 8; ++k)
            if (tr[c * 16 + k] >= t0) fprintf(f, "%d %d %llu\n", c, k, tr[c * 16 + k] - t0);
        fclose(f);
      }
      CK(cudaMemset(inst->gu_trace, 0, sizeof(unsigned long long) * tr.size()));
    }
    if (inst->gu_sk && *inst->h_gu_err) {
      inst->err = "decode gate/up stream-K: a partial-tile wait timed out (CTAs not co-resident; ECOSERVE_GU_SK=0 "
                  "disables it)";
      inst->dead = true;
      return ECOSERVE_ERR_CUDA;
    }
    if (inst->flow && *inst->h_flow_err) {
      inst->err = "decode flow: a dependency wait timed out (CTAs not co-resident; ECOSERVE_FLOW=0 disables it)";
      inst->dead = true;
      return ECOSERVE_ERR_CUDA;
    }
    if (inst->chain && *inst->h_chain_err) {
      inst->err = "decode chain: grid barrier timed out (CTAs not co-resident; set ECOSERVE_CHAIN=0 when several "
                  "instances share a GPU)";
      inst->dead = true;
      return ECOSERVE_ERR_CUDA;
    }
    if (host_timing_enabled()) {
      const auto t_sync = std::chrono::steady_clock::now();
      fprintf(stderr, "[ecoserve] decode step B=%d: host enqueue %.1f us, enqueue+gpu %.1f us\n", B,
              std::chrono::duration<double, std::micro>(t_enq1 - t_enq0).count(),
              std::chrono::duration<double, std::micro>(t_sync - t_enq0).count());
    }
    inst->prof.resolve();
    inst->prof.tokens[1] += B;
    inst->prof.h2d += sizeof(int) * used;
    inst->prof.d2h += sizeof(int) * B;
    if (ecoserve_status ts = check_tokens(inst, B); ts != ECOSERVE_OK) return ts;
    for (int k = 0; k < B; ++k) {
      Req* r = rs[live[k]];
      r->last_token = inst->h_tokens[k];
      r->n_gen += 1;
      r->finished = r->n_gen >= r->max_new;
      tokens[(int64_t)live[k] * steps + s] = r->last_token;
    }
  }
  if (n_finished) {
    int c = 0;
    for (int i = 0; i < n; ++i) c += rs[i]->finished ? 1 : 0;
    *n_finished = c;
  }
  return ECOSERVE_OK;
}

// Direct NVLink copies for a buffer on another GPU: enable peer access from this
// instance's device (without it, cross-device cudaMemcpyAsync is staged through the host).
static void enable_peer_for(int dev, const void* ptr) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if (at.type != cudaMemoryTypeDevice || at.device == dev) return;
  int ok = 0;
  if (cudaDeviceCanAccessPeer(&ok, dev, at.device) == cudaSuccess && ok) {
    if (cudaDeviceEnablePeerAccess(at.device, 0) != cudaSuccess) cudaGetLastError();  // already enabled is fine
  }
}

ecoserve_status ecoserve_kv_export(ecoserve_instance* inst, int64_t req_id, void* dst, int64_t dst_bytes,
                                   int32_t* prompt, int32_t prompt_cap, ecoserve_req_state* state) {
  if (!inst || !dst || !state) return ECOSERVE_ERR_INVALID_ARG;
  if (inst->dead) return ECOSERVE_ERR_CUDA;
  auto it = inst->reqs.find(req_id);
  if (it == inst->reqs.end() || it->second.n_gen < 1) return ECOSERVE_ERR_STATE;
  const Req& r = it->second;
  const int64_t bb = inst->blk_stride * (int64_t)sizeof(bf16);
  if (dst_bytes < bb * (int64_t)r.blocks.size() || (prompt && prompt_cap < r.S)) return ECOSERVE_ERR_INVALID_ARG;
  CK(cudaSetDevice(inst->device));
  enable_peer_for(inst->device, dst);
  for (size_t b = 0; b < r.blocks.size(); ++b)  // one contiguous span per block (all layers, K and V)
    CK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(dst) + b * bb, inst->pool + (int64_t)r.blocks[b] * inst->blk_stride,
                       bb, cudaMemcpyDefault, inst->stream));
  CK(cudaStreamSynchronize(inst->stream));
  if (prompt) memcpy(prompt, r.prompt.data(), sizeof(int32_t) * r.S);
  state->req_id = r.id;
  state->prompt_len = r.S;
  state->max_new_tokens = r.max_new;
  state->n_generated = r.n_gen;
  state->last_token = r.last_token;
  state->n_blocks = (int32_t)r.blocks.size();
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_kv_import(ecoserve_instance* inst, const ecoserve_req_state* st, const int32_t* prompt,
                                   const void* src) {
  if (!inst || !st || !prompt || !src || st->prompt_len < 1 || st->n_generated < 1 || st->n_blocks < 0)
    return ECOSERVE_ERR_INVALID_ARG;
  if (inst->dead) return ECOSERVE_ERR_CUDA;
  const int64_t kv_len = (int64_t)st->prompt_len + st->n_generated - 1;  // tokens whose K/V are stored
  if (st->n_blocks != (int)((kv_len + BLOCK - 1) / BLOCK) || st->prompt_len + st->max_new_tokens > inst->P_max)
    return ECOSERVE_ERR_INVALID_ARG;
  if (inst->reqs.count(st->req_id)) return ECOSERVE_ERR_STATE;
  if ((int64_t)inst->free_blocks.size() < st->n_blocks) return ECOSERVE_ERR_KV_EXHAUSTED;
  CK(cudaSetDevice(inst->device));
  enable_peer_for(inst->device, src);
  Req r;
  r.id = st->req_id;
  r.S = st->prompt_len;
  r.max_new = st->max_new_tokens;
  r.n_gen = st->n_generated;
  r.last_token = st->last_token;
  r.prefilled = r.S;
  r.finished = r.n_gen >= r.max_new;
  r.prompt.assign(prompt, prompt + r.S);
  const int64_t bb = inst->blk_stride * (int64_t)sizeof(bf16);
  for (int b = 0; b < st->n_blocks; ++b) {
    r.blocks.push_back(inst->free_blocks.back());
    inst->free_blocks.pop_back();
  }
  for (int b = 0; b < st->n_blocks; ++b)
    CK(cudaMemcpyAsync(inst->pool + (int64_t)r.blocks[b] * inst->blk_stride,
                       reinterpret_cast<const uint8_t*>(src) + b * bb, bb, cudaMemcpyDefault, inst->stream));
  CK(cudaStreamSynchronize(inst->stream));
  inst->reqs[r.id] = std::move(r);
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_set_profiling(ecoserve_instance* inst, int32_t level) {
  if (!inst || level < 0 || level > 2) return ECOSERVE_ERR_INVALID_ARG;
  inst->prof.level = level;
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_get_timing(ecoserve_instance* inst, ecoserve_timing* out, int32_t reset) {
  if (!inst || !out) return ECOSERVE_ERR_INVALID_ARG;
  const Prof& p = inst->prof;
  memset(out, 0, sizeof(*out));
  out->prefill_ms = p.ms[P_PREFILL];
  out->decode_ms = p.ms[P_DECODE];
  out->prefill_tokens = p.tokens[0];
  out->decode_tokens = p.tokens[1];
  out->launches = p.launches;
  out->gemm_prefill_ms = p.ms[P_GEMM_PREFILL];
  out->gemm_prefill_flop = p.work[P_GEMM_PREFILL];
  out->gemm_prefill_launches = p.count[P_GEMM_PREFILL];
  out->gemm_decode_ms = p.ms[P_GEMM_DECODE];
  out->gemm_decode_bytes = p.work[P_GEMM_DECODE];
  out->gemm_decode_launches = p.count[P_GEMM_DECODE];
  out->attn_prefill_ms = p.ms[P_ATTN_PREFILL];
  out->attn_prefill_flop = p.work[P_ATTN_PREFILL];
  out->attn_prefill_launches = p.count[P_ATTN_PREFILL];
  out->attn_decode_ms = p.ms[P_ATTN_DECODE];
  out->attn_decode_bytes = p.work[P_ATTN_DECODE];
  out->attn_decode_launches = p.count[P_ATTN_DECODE];
  out->other_ms = p.ms[P_OTHER];
  out->other_launches = p.count[P_OTHER];
  out->h2d_bytes = p.h2d;
  out->d2h_bytes = p.d2h;
  if (reset) inst->prof.reset();
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_release(ecoserve_instance* inst, const int64_t* req_ids, int32_t n) {
  if (!inst || n < 0 || (n > 0 && !req_ids)) return ECOSERVE_ERR_INVALID_ARG;
  for (int i = 0; i < n; ++i)
    if (!inst->reqs.count(req_ids[i])) return ECOSERVE_ERR_STATE;
  for (int i = 0; i < n; ++i) {
    auto it = inst->reqs.find(req_ids[i]);
    for (int b : it->second.blocks) inst->free_blocks.push_back(b);
    inst->reqs.erase(it);
  }
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_get_status(const ecoserve_instance* inst, ecoserve_instance_status* out,
                                    ecoserve_req_status* reqs, int32_t cap) {
  if (!inst || !out || cap < 0 || (cap > 0 && !reqs)) return ECOSERVE_ERR_INVALID_ARG;
  out->alive = inst->dead ? 0 : 1;
  out->n_requests = (int32_t)inst->reqs.size();
  out->blocks_total = inst->num_blocks;
  out->blocks_used = inst->num_blocks - (int64_t)inst->free_blocks.size();
  int k = 0;
  for (auto& kvp : inst->reqs) {
    if (k >= cap) break;
    const Req& r = kvp.second;
    reqs[k].req_id = r.id;
    reqs[k].prompt_len = r.S;
    reqs[k].n_generated = r.n_gen;
    reqs[k].finished = r.finished ? 1 : 0;
    reqs[k].n_blocks = (int32_t)r.blocks.size();
    ++k;
  }
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_debug_hidden(ecoserve_instance* inst, int64_t req_id, int32_t layer, float* out) {
  if (!inst || !out || layer < 0 || layer > inst->L) return ECOSERVE_ERR_INVALID_ARG;
  if (!inst->debug) return ECOSERVE_ERR_UNSUPPORTED;
  auto it = inst->dbg_rows.find(req_id);
  if (it == inst->dbg_rows.end()) return ECOSERVE_ERR_STATE;
  const float* src = inst->dbg + ((int64_t)layer * inst->T_max + it->second.first) * inst->H;
  CK(cudaMemcpy(out, src, sizeof(float) * (int64_t)it->second.second * inst->H, cudaMemcpyDeviceToHost));
  return ECOSERVE_OK;
}

ecoserve_status ecoserve_debug_force_token(ecoserve_instance* inst, int64_t req_id, int32_t token) {
  if (!inst || token < 0 || token >= inst->V) return ECOSERVE_ERR_INVALID_ARG;
  if (!inst->debug) return ECOSERVE_ERR_UNSUPPORTED;
  auto it = inst->reqs.find(req_id);
  if (it == inst->reqs.end() || it->second.n_gen < 1 || it->second.finished) return ECOSERVE_ERR_STATE;
  it->second.last_token = token;
  return ECOSERVE_OK;
}

}  // extern "C"
