// extern "C" boundary of libkvrot_b200.so: validation, dispatch, error text.
// See include/kvrot_b200.h for the contract and the reference interface each
// entry point replaces.
#include <cstdarg>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <new>
#include <mutex>
#include <vector>

#include "kvr_common.cuh"
#include "kvr_internal.h"

using namespace kvr;

static thread_local char g_err[512] = "";

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

static int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(KVR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return KVR_OK;
}

static bool pow2(int x) { return x >= 1 && (x & (x - 1)) == 0; }

static int check_order(int d, int order) {
  if (!pow2(order)) return fail(KVR_ERR_ORDER, "order=%d is not a power of two", order);
  if (d % order != 0) return fail(KVR_ERR_ORDER, "order=%d does not divide dim=%d", order, d);
  return KVR_OK;
}

static int make_signs(const uint32_t* words, int d, Signs& s, int& has) {
  memset(&s, 0, sizeof(s));
  has = words != nullptr;
  if (!has) return KVR_OK;
  if (d > KVR_MAX_HEAD_DIM) return fail(KVR_ERR_UNSUPPORTED, "signs for head_dim %d > %d", d, KVR_MAX_HEAD_DIM);
  memcpy(s.w, words, sizeof(uint32_t) * ((d + 31) / 32));
  return KVR_OK;
}

static int to_pool(const kvr_pool* in, Pool& p) {
  if (!in || !in->base) return fail(KVR_ERR_ARG, "null pool");
  p.base = reinterpret_cast<uint8_t*>(in->base);
  p.num_pages = in->num_pages;
  p.P = in->page_tokens;
  p.H = in->num_kv_heads;
  p.d = in->head_dim;
  p.page_bytes = in->page_bytes;
  p.T = in->cell_tokens;
  p.cell_bytes = in->cell_bytes;
  p.prec = in->precision;
  if (p.prec != KVR_PREC_INT4 && p.prec != KVR_PREC_BF16) return fail(KVR_ERR_ARG, "bad pool precision %d", p.prec);
  const int64_t need = p.prec == KVR_PREC_BF16 ? 4LL * p.T * p.d : (int64_t)p.T * (p.d + 10);
  if (p.T < 1 || p.P % p.T != 0 || p.cell_bytes < need)
    return fail(KVR_ERR_SHAPE, "inconsistent pool geometry (P=%d, T=%d, cell=%d)", p.P, p.T, p.cell_bytes);
  return KVR_OK;
}

CUresult kvr_encode_tensor_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows,
                                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_rows,
                                  CUtensorMapSwizzle swz) {
  typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static encode_fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return CUDA_ERROR_NOT_FOUND;
    fn = reinterpret_cast<encode_fn>(f);
  }
  const cuuint64_t dims[2] = {inner, rows < 1 ? 1 : rows};
  const cuuint64_t strides[1] = {row_stride_bytes};
  const cuuint32_t box[2] = {box_inner, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

int kvr_current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (dev >= 0 && dev < KVR_MAX_DEVICES) ? dev : KVR_MAX_DEVICES - 1;
}

// SM count of the calling thread's current device (cached per device: one process
// may drive several GPUs)
int kvr_num_sms() {
  static int sms[KVR_MAX_DEVICES];
  static bool known[KVR_MAX_DEVICES];
  const int dev = kvr_current_device();
  if (!known[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    sms[dev] = n;
    known[dev] = true;
  }
  return sms[dev];
}

static std::mutex g_pw_mu;
static std::vector<cudaStream_t> g_pw;  // streams whose last pool access was a write

void kvr_mark_pool_written(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_pw_mu);
  for (cudaStream_t x : g_pw)
    if (x == st) return;
  g_pw.push_back(st);
}

bool kvr_take_pool_written(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_pw_mu);
  for (size_t i = 0; i < g_pw.size(); ++i)
    if (g_pw[i] == st) {
      g_pw[i] = g_pw.back();
      g_pw.pop_back();
      return true;
    }
  return false;
}

static int decode_step_impl(const void* q, int32_t q_dtype, const void* new_k, const void* new_v, int32_t kv_dtype,
                            const int64_t* new_slot, const kvr_pool* pool, const int32_t* block_table,
                            int32_t bt_stride, const int32_t* seq_lens, int32_t batch, int32_t num_q_heads,
                            int32_t max_seq_len, int32_t rot_order, int32_t rotate, int32_t targets,
                            const uint32_t* sign_words, float* out, void* workspace, size_t workspace_bytes,
                            int32_t num_splits, uint32_t* flags, void* stream, int q_host_staged);

extern "C" {

const char* kvr_last_error(void) { return g_err; }
void kvr_note_pool_write(void* stream) { kvr_mark_pool_written((cudaStream_t)stream); }
void kvr_debug_decode_trace(void* trace) { kvr_set_decode_trace(trace); }
void kvr_debug_set_k1_impl(int32_t impl) { kvr_set_k1_impl(impl); }
int kvr_abi_version(void) { return KVR_ABI_VERSION; }

// Host-side validation helper (not a compute path): 1 when all n values at host
// pointer `p` are finite, 0 otherwise, -1 for a bad dtype.  Lets the serving step
// reject NaN/Inf inputs before it commits any allocator state (cache.py:225-233).
int kvr_host_all_finite(const void* p, int32_t dtype, int64_t n) {
  if (n <= 0) return 1;
  if (!p) return -1;
  uint32_t bad = 0u;
  switch (dtype) {
    case KVR_BF16:    // exponent all ones
    case KVR_F16: {   // four 16-bit values per 64-bit word: a lane with the exponent mask all set
      const uint64_t m = dtype == KVR_BF16 ? 0x7F807F807F807F80ull : 0x7C007C007C007C00ull;
      const uint16_t* u = static_cast<const uint16_t*>(p);
      int64_t i = 0;
      if (!(reinterpret_cast<uintptr_t>(p) & 7)) {
        const uint64_t* w = static_cast<const uint64_t*>(p);
        uint64_t acc = 0;
        for (; i + 4 <= n; i += 4) {
          const uint64_t x = (w[i >> 2] & m) ^ m;  // 16-bit lane == 0 <=> non-finite
          acc |= (x - 0x0001000100010001ull) & ~x & 0x8000800080008000ull;
        }
        bad |= acc != 0;
      }
      const uint16_t e = (uint16_t)(m & 0xFFFF);
      for (; i < n; ++i) bad |= ((u[i] & e) == e);
      return bad ? 0 : 1;
    }
    case KVR_F32: {
      const uint32_t* u = static_cast<const uint32_t*>(p);
      for (int64_t i = 0; i < n; ++i) bad |= ((u[i] & 0x7F800000u) == 0x7F800000u);
      return bad ? 0 : 1;
    }
    case KVR_F64: {
      const uint64_t* u = static_cast<const uint64_t*>(p);
      for (int64_t i = 0; i < n; ++i) bad |= ((u[i] & 0x7FF0000000000000ull) == 0x7FF0000000000000ull);
      return bad ? 0 : 1;
    }
  }
  return -1;
}
int kvr_device_sms(void) { return kvr_num_sms(); }

// ---- DecodePlan.step's per-step host work in two calls (Python keeps only the
// allocator bookkeeping between them)
static int host_finite_bytes(const void* p, int32_t dtype, int64_t n) { return kvr_host_all_finite(p, dtype, n); }

int kvr_step_stage(void* ring_event, void* staging, const void* q, int64_t q_off, int64_t q_bytes, int32_t q_dtype,
                   const void* k, int64_t k_off, const void* v, int64_t v_off, int64_t kv_bytes, int32_t kv_dtype,
                   int32_t check) {
  if (!staging) return fail(KVR_ERR_ARG, "step_stage: null staging buffer");
  if (ring_event && cudaEventSynchronize((cudaEvent_t)ring_event) != cudaSuccess)
    return fail(KVR_ERR_CUDA, "step_stage: cudaEventSynchronize failed");
  const int esz[] = {8, 4, 2, 2};  // KVR_F64, F32, BF16, F16
  if (check) {
    if (q && q_dtype >= KVR_F64 && q_dtype <= KVR_F16 && host_finite_bytes(q, q_dtype, q_bytes / esz[q_dtype]) != 1)
      return 0;
    if (kv_dtype >= KVR_F64 && kv_dtype <= KVR_F16) {
      if (k && host_finite_bytes(k, kv_dtype, kv_bytes / esz[kv_dtype]) != 1) return 0;
      if (v && host_finite_bytes(v, kv_dtype, kv_bytes / esz[kv_dtype]) != 1) return 0;
    }
  }
  uint8_t* st = static_cast<uint8_t*>(staging);
  if (q) memcpy(st + q_off, q, (size_t)q_bytes);
  if (k) memcpy(st + k_off, k, (size_t)kv_bytes);
  if (v) memcpy(st + v_off, v, (size_t)kv_bytes);
  return 1;
}

// A pinned staging ring bound to fixed host inputs and captured graphs: one call per step.
struct kvr_step_ring {
  void* q;
  void* k;
  void* v;
  int64_t q_off, q_bytes, k_off, v_off, kv_bytes, meta_bytes, bytes;
  int32_t q_dtype, kv_dtype, check, n;
  void* stream;
  void* copy_stream;  // non-NULL: the copy goes on this stream and `stream` waits for it (copy_event)
  void* copy_event[16];
  // direct mode (kvr_step_ring_set_decode): each run launches the fused decode step itself, its
  // inputs read by the kernel from the pinned staging slot (no graph, no stage-in copy)
  int direct;
  int32_t d_q_dtype, d_kv_dtype, d_bt_stride, d_batch, d_nq, d_max_len, d_rot_order, d_rotate, d_targets, d_splits,
      d_has_signs;
  kvr_pool d_pool;
  const int32_t* d_bt;
  uint32_t d_signs[KVR_MAX_HEAD_DIM / 32];
  float* d_out;
  void* d_ws;
  size_t d_ws_bytes;
  uint32_t* d_flags;
  void* staging[16];
  void* dev[16];
  void* exec[16];
  void* event[16];
};

kvr_step_ring* kvr_step_ring_create(int32_t n_slots, const void* q, int64_t q_off, int64_t q_bytes, int32_t q_dtype,
                                    const void* k, int64_t k_off, const void* v, int64_t v_off, int64_t kv_bytes,
                                    int32_t kv_dtype, int64_t meta_bytes, int64_t bytes, int32_t check, void* stream) {
  if (n_slots < 1 || n_slots > 16) {
    fail(KVR_ERR_ARG, "step_ring_create: 1..16 slots");
    return nullptr;
  }
  kvr_step_ring* r = new (std::nothrow) kvr_step_ring();
  if (!r) return nullptr;
  r->q = const_cast<void*>(q);
  r->k = const_cast<void*>(k);
  r->v = const_cast<void*>(v);
  r->q_off = q_off;
  r->q_bytes = q_bytes;
  r->k_off = k_off;
  r->v_off = v_off;
  r->kv_bytes = kv_bytes;
  r->q_dtype = q_dtype;
  r->kv_dtype = kv_dtype;
  r->meta_bytes = meta_bytes;
  r->bytes = bytes;
  r->check = check;
  r->n = n_slots;
  r->stream = stream;
  return r;
}

int kvr_step_ring_set_slot(kvr_step_ring* r, int32_t i, void* staging, void* dev, void* graph_exec, void* event) {
  if (!r || i < 0 || i >= r->n) return fail(KVR_ERR_ARG, "step_ring_set_slot: bad ring or slot");
  r->staging[i] = staging;
  r->dev[i] = dev;
  r->exec[i] = graph_exec;
  r->event[i] = event;
  return KVR_OK;
}

void kvr_step_ring_destroy(kvr_step_ring* r) {
  if (!r) return;
  for (int i = 0; i < 16; ++i)
    if (r->copy_event[i]) cudaEventDestroy((cudaEvent_t)r->copy_event[i]);
  delete r;
}

int kvr_step_ring_set_decode(kvr_step_ring* r, int32_t q_dtype, int32_t kv_dtype, const kvr_pool* pool,
                             const int32_t* block_table, int32_t bt_stride, int32_t batch, int32_t num_q_heads,
                             int32_t max_seq_len, int32_t rot_order, int32_t rotate, int32_t targets,
                             const uint32_t* sign_words, float* out, void* workspace, size_t workspace_bytes,
                             int32_t num_splits, uint32_t* flags, int32_t mode) {
  if (!r || !pool) return fail(KVR_ERR_ARG, "step_ring_set_decode: null ring / pool");
  if (mode < 1 || mode > 2) return fail(KVR_ERR_ARG, "step_ring_set_decode: mode 1 or 2");
  r->d_q_dtype = q_dtype;
  r->d_kv_dtype = kv_dtype;
  r->d_pool = *pool;
  r->d_bt = block_table;
  r->d_bt_stride = bt_stride;
  r->d_batch = batch;
  r->d_nq = num_q_heads;
  r->d_max_len = max_seq_len;
  r->d_rot_order = rot_order;
  r->d_rotate = rotate;
  r->d_targets = targets;
  r->d_has_signs = sign_words != nullptr;
  if (sign_words) memcpy(r->d_signs, sign_words, sizeof(r->d_signs[0]) * ((pool->head_dim + 31) / 32));
  r->d_out = out;
  r->d_ws = workspace;
  r->d_ws_bytes = workspace_bytes;
  r->d_splits = num_splits;
  r->d_flags = flags;
  r->direct = mode;
  return KVR_OK;
}

static double g_ring_ns[4];
static long g_ring_calls;
static inline double now_ns() {
  return (double)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
void kvr_debug_step_ring_times(double* out4) {  // profiling aid: mean ns per run (stage, meta, launch, record)
  for (int k = 0; k < 4; ++k) out4[k] = g_ring_calls ? g_ring_ns[k] / g_ring_calls : 0.0;
}
int kvr_step_ring_run(kvr_step_ring* r, int32_t i, const void* meta) {
  if (!r || i < 0 || i >= r->n || !(r->exec[i] || r->direct)) return fail(KVR_ERR_ARG, "step_ring_run: bad ring or slot");
  const double t0 = now_ns();
  ++g_ring_calls;
  const int rc = kvr_step_stage(r->event[i], r->staging[i], r->q, r->q_off, r->q_bytes, r->q_dtype, r->k, r->k_off,
                                r->v, r->v_off, r->kv_bytes, r->kv_dtype, r->check);
  if (rc != 1) return rc == 0 ? KVR_ERR_NONFINITE : rc;
  const double t1 = now_ns();
  g_ring_ns[0] += t1 - t0;
  memcpy(r->staging[i], meta, (size_t)r->meta_bytes);
  if (r->direct) {  // slot ids | lengths | q | k | v all in the pinned slot: the kernel reads them in place
    uint8_t* st = static_cast<uint8_t*>(r->staging[i]);
    const int B = r->d_batch;
    const uint8_t* in = st;  // where the kernel reads q / k / v
    int q_staged = 1;
    if (r->direct == 2) {
      // the slot (ids, lengths, q, k, v) goes to its device twin through a one-CTA copy kernel chained
      // in front of the decode: the copy overlaps the previous step; the decode reads it all after its
      // grid-dependency wait (pinned-memory reads in its prologue cost ~12 us a step, measured)
      if (int e = kvr_launch_stage_copy(r->dev[i], st, r->bytes, (cudaStream_t)r->stream))
        return fail(e, "step_ring_run: stage copy launch failed");
      in = static_cast<const uint8_t*>(r->dev[i]);
      q_staged = 2;  // slot ids / lengths too come from the copy: the decode reads them after its wait
    }
    const uint8_t* meta_in = r->direct == 2 ? in : st;
    const double t2 = now_ns();
    g_ring_ns[1] += t2 - t1;
    if (int e = decode_step_impl(in + r->q_off, r->d_q_dtype, in + r->k_off, in + r->v_off, r->d_kv_dtype,
                                 reinterpret_cast<const int64_t*>(meta_in), &r->d_pool, r->d_bt, r->d_bt_stride,
                                 reinterpret_cast<const int32_t*>(meta_in + 8 * B), B, r->d_nq, r->d_max_len,
                                 r->d_rot_order, r->d_rotate, r->d_targets, r->d_has_signs ? r->d_signs : nullptr,
                                 r->d_out, r->d_ws, r->d_ws_bytes, r->d_splits, r->d_flags, r->stream, q_staged))
      return e;
    const double t3 = now_ns();
    g_ring_ns[2] += t3 - t2;
    if (cudaEventRecord((cudaEvent_t)r->event[i], (cudaStream_t)r->stream) != cudaSuccess)
      return fail(KVR_ERR_CUDA, "step_ring_run: cudaEventRecord failed");
    g_ring_ns[3] += now_ns() - t3;
    return KVR_OK;
  }
  if (!r->copy_stream) return kvr_step_launch(r->dev[i], r->staging[i], r->bytes, r->exec[i], r->event[i], r->stream);
  // side-stream copy: it may overlap the previous step's kernel (the slot's last reader is done)
  cudaStream_t cs = (cudaStream_t)r->copy_stream, st = (cudaStream_t)r->stream;
  if (cudaMemcpyAsync(r->dev[i], r->staging[i], (size_t)r->bytes, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
      cudaEventRecord((cudaEvent_t)r->copy_event[i], cs) != cudaSuccess ||
      cudaStreamWaitEvent(st, (cudaEvent_t)r->copy_event[i], 0) != cudaSuccess)
    return fail(KVR_ERR_CUDA, "step_ring_run: side-stream copy failed");
  return kvr_step_launch(nullptr, nullptr, 0, r->exec[i], r->event[i], r->stream);
}

int kvr_step_ring_set_copy_stream(kvr_step_ring* r, void* copy_stream) {
  if (!r) return fail(KVR_ERR_ARG, "step_ring_set_copy_stream: null ring");
  if (copy_stream)
    for (int i = 0; i < r->n; ++i)
      if (!r->copy_event[i] &&
          cudaEventCreateWithFlags((cudaEvent_t*)&r->copy_event[i], cudaEventDisableTiming) != cudaSuccess)
        return fail(KVR_ERR_CUDA, "step_ring_set_copy_stream: cudaEventCreate failed");
  r->copy_stream = copy_stream;
  return KVR_OK;
}

int kvr_step_launch(void* dev_buf, const void* staging, int64_t bytes, void* graph_exec, void* ring_event,
                    void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (bytes > 0 && cudaMemcpyAsync(dev_buf, staging, (size_t)bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return fail(KVR_ERR_CUDA, "step_launch: cudaMemcpyAsync failed");
  if (graph_exec && cudaGraphLaunch((cudaGraphExec_t)graph_exec, st) != cudaSuccess)
    return fail(KVR_ERR_CUDA, "step_launch: cudaGraphLaunch failed");
  if (ring_event && cudaEventRecord((cudaEvent_t)ring_event, st) != cudaSuccess)
    return fail(KVR_ERR_CUDA, "step_launch: cudaEventRecord failed");
  return KVR_OK;
}

int kvr_pool_init(kvr_pool* pool, void* base, int64_t num_pages, int32_t page_tokens, int32_t num_kv_heads,
                  int32_t head_dim) {
  if (!pool) return fail(KVR_ERR_ARG, "null pool");
  if (page_tokens < 1 || num_kv_heads < 1 || head_dim < 2 || (head_dim & 1) || num_pages < 0)
    return fail(KVR_ERR_SHAPE, "bad pool geometry P=%d H=%d d=%d", page_tokens, num_kv_heads, head_dim);
  const int T = (page_tokens % 16 == 0) ? 16 : page_tokens;
  pool->base = base;
  pool->num_pages = num_pages;
  pool->page_tokens = page_tokens;
  pool->num_kv_heads = num_kv_heads;
  pool->head_dim = head_dim;
  pool->cell_tokens = T;
  pool->cell_bytes = (T * (head_dim + 10) + 15) & ~15;
  pool->precision = KVR_PREC_INT4;
  const int64_t pb = (int64_t)num_kv_heads * (page_tokens / T) * pool->cell_bytes;
  if (pb > 0x7fffffff) return fail(KVR_ERR_SHAPE, "page too large");
  pool->page_bytes = (int32_t)pb;
  return KVR_OK;
}

int kvr_pool_init_bf16(kvr_pool* pool, void* base, int64_t num_pages, int32_t page_tokens, int32_t num_kv_heads,
                       int32_t head_dim) {
  if (int rc = kvr_pool_init(pool, base, num_pages, page_tokens, num_kv_heads, head_dim)) return rc;
  pool->precision = KVR_PREC_BF16;
  pool->cell_bytes = 4 * pool->cell_tokens * head_dim;  // head_dim even -> 16-B multiple when T * d % 4 == 0
  const int64_t pb = (int64_t)num_kv_heads * (page_tokens / pool->cell_tokens) * pool->cell_bytes;
  if (pb > 0x7fffffff) return fail(KVR_ERR_SHAPE, "page too large");
  pool->page_bytes = (int32_t)pb;
  return KVR_OK;
}

int kvr_fwht_rows_f64(double* x, int64_t n, int32_t d, int32_t order, void* stream) {
  if (n < 0 || d < 1) return fail(KVR_ERR_SHAPE, "bad shape (%lld, %d)", (long long)n, d);
  if (int rc = check_order(d, order)) return rc;
  if (n == 0 || order == 1) return KVR_OK;
  if (!x) return fail(KVR_ERR_ARG, "null x");
  if (d > 6144) return fail(KVR_ERR_UNSUPPORTED, "dim %d > 6144", d);
  kvr_launch_fwht_f64(x, n, d, order, (cudaStream_t)stream);
  return check_launch("fwht_rows_f64");
}

int kvr_pack_rows(const uint8_t* nibbles, uint8_t* out, int64_t n, int32_t d, void* stream) {
  if (n < 0 || d < 0 || (d & 1)) return fail(KVR_ERR_SHAPE, "pack_rows needs even d, got %d", d);
  if (n == 0 || d == 0) return KVR_OK;
  kvr_launch_pack(nibbles, out, n, d, (cudaStream_t)stream);
  return check_launch("pack_rows");
}

int kvr_unpack_rows(const uint8_t* packed, uint8_t* out, int64_t n, int32_t logical_len, void* stream) {
  if (n < 0 || logical_len < 0 || (logical_len & 1))
    return fail(KVR_ERR_SHAPE, "unpack_rows needs even logical_len, got %d", logical_len);
  if (n == 0 || logical_len == 0) return KVR_OK;
  kvr_launch_unpack(packed, out, n, logical_len, (cudaStream_t)stream);
  return check_launch("unpack_rows");
}

int kvr_quantize_rows_f64(const double* x, int64_t n, int32_t d, uint8_t* packed, float* scale, uint8_t* zp,
                          void* stream) {
  if (n < 0 || d < 2 || (d & 1)) return fail(KVR_ERR_SHAPE, "expected (n, even d) rows, got d=%d", d);
  if (n == 0) return KVR_OK;
  if (d > 6144) return fail(KVR_ERR_UNSUPPORTED, "dim %d > 6144", d);
  kvr_launch_quantize_f64(x, n, d, packed, scale, zp, (cudaStream_t)stream);
  return check_launch("quantize_rows_f64");
}

int kvr_dequantize_rows_f64(const uint8_t* packed, const float* scale, const uint8_t* zp, int64_t n,
                            int32_t logical_len, double* out, void* stream) {
  if (n < 0 || logical_len < 0 || (logical_len & 1)) return fail(KVR_ERR_SHAPE, "bad logical_len %d", logical_len);
  if (n == 0 || logical_len == 0) return KVR_OK;
  kvr_launch_dequantize_f64(packed, scale, zp, n, logical_len, out, (cudaStream_t)stream);
  return check_launch("dequantize_rows_f64");
}

int kvr_block_rotate(const void* x, int32_t in_dtype, void* out, int32_t out_dtype, int64_t n, int32_t d,
                     int32_t order, const uint32_t* sign_words, int32_t inverse, void* stream) {
  if (n < 0 || d < 1) return fail(KVR_ERR_SHAPE, "bad shape");
  if (int rc = check_order(d, order)) return rc;
  if (d > 6144) return fail(KVR_ERR_UNSUPPORTED, "dim %d > 6144", d);
  Signs s;
  int has;
  if (int rc = make_signs(sign_words, d, s, has)) return rc;
  if (n == 0) return KVR_OK;
  int rc = kvr_launch_block_rotate(x, in_dtype, out, out_dtype, n, d, order, s, has, inverse, (cudaStream_t)stream);
  if (rc) return fail(rc, "block_rotate: unsupported dtype combination (%d -> %d)", in_dtype, out_dtype);
  return check_launch("block_rotate");
}

int kvr_rows_matmul_f64(const void* x, int32_t in_dtype, const double* m, void* y, int32_t out_dtype, int64_t n,
                        int32_t d, void* stream) {
  if (n < 0 || d < 1) return fail(KVR_ERR_SHAPE, "rows_matmul: bad shape (n=%lld, d=%d)", (long long)n, d);
  if (d > 768) return fail(KVR_ERR_UNSUPPORTED, "rows_matmul: dim %d > 768", d);
  if (n == 0) return KVR_OK;
  if (!x || !m || !y) return fail(KVR_ERR_ARG, "rows_matmul: null pointer");
  if (x == y) return fail(KVR_ERR_ARG, "rows_matmul: in-place (x == y) is not supported");
  int rc = kvr_launch_rows_matmul(x, in_dtype, m, y, out_dtype, n, d, (cudaStream_t)stream);
  if (rc) return fail(rc, "rows_matmul: unsupported dtype combination (%d -> %d)", in_dtype, out_dtype);
  return check_launch("rows_matmul_f64");
}

int kvr_rotate_quantize_store(const void* k, const void* v, int32_t in_dtype, int64_t n_tok,
                              const int64_t* slot_mapping, const kvr_pool* pool, int32_t rot_order, int32_t rotate,
                              int32_t targets, const uint32_t* sign_words, int32_t exact, uint32_t* flags,
                              void* stream) {
  Pool pl;
  if (int rc = to_pool(pool, pl)) return rc;
  if (n_tok < 0) return fail(KVR_ERR_SHAPE, "n_tok < 0");
  if (n_tok == 0) return KVR_OK;
  if (!k || !v || !slot_mapping) return fail(KVR_ERR_ARG, "null k/v/slot_mapping");
  if (in_dtype < KVR_F64 || in_dtype > KVR_F16) return fail(KVR_ERR_ARG, "bad dtype %d", in_dtype);
  if (rotate) {
    if (int rc = check_order(pl.d, rot_order)) return rc;
  } else {
    rot_order = 1;
  }
  Signs s;
  int has;
  if (int rc = make_signs(rotate ? sign_words : nullptr, pl.d, s, has)) return rc;
  const int rot_k = rotate ? 1 : 0;
  const int rot_v = (rotate && targets == KVR_KEYS_AND_VALUES) ? 1 : 0;
  cudaStream_t st = (cudaStream_t)stream;
  kvr_mark_pool_written(st);  // a decode launched next on this stream must not prefetch before its wait
  if (pl.prec == KVR_PREC_BF16) {  // raw vectors, rotation ignored (cache.py:264-266)
    if (int rc = kvr_launch_store_bf16(k, v, in_dtype, n_tok, slot_mapping, pl, flags, st))
      return fail(rc, "rotate_quantize_store (bf16 pool): launch failed (%d)", rc);
    return check_launch("rotate_quantize_store");
  }
  int rc = KVR_ERR_UNSUPPORTED;
  if (!exact) rc = kvr_launch_store_fast(k, v, in_dtype, n_tok, slot_mapping, pl, rot_order, rot_k, rot_v, s, has,
                                         flags, st);
  if (rc == KVR_ERR_UNSUPPORTED) {
    if (pl.d > 6144) return fail(KVR_ERR_UNSUPPORTED, "dim %d > 6144", pl.d);
    rc = kvr_launch_store_exact(k, v, in_dtype, n_tok, slot_mapping, pl, rot_order, rot_k, rot_v, s, has, flags, st);
  }
  if (rc) return fail(rc, "rotate_quantize_store: launch failed (%d)", rc);
  return check_launch("rotate_quantize_store");
}

int kvr_rotate_quantize_store_learned(const void* k, const void* v, int32_t in_dtype, int64_t n_tok,
                                      const int64_t* slot_mapping, const kvr_pool* pool, int32_t rot_order,
                                      int32_t targets, int32_t learned_values, const uint32_t* sign_words,
                                      const void* t_img, const double* r_t, uint32_t* flags, void* stream) {
  Pool pl;
  if (int rc = to_pool(pool, pl)) return rc;
  if (n_tok < 0) return fail(KVR_ERR_SHAPE, "n_tok < 0");
  if (!k || !v || !slot_mapping || !t_img || !r_t) return fail(KVR_ERR_ARG, "null k/v/slot_mapping/t_img/r_t");
  if (in_dtype < KVR_F64 || in_dtype > KVR_F16) return fail(KVR_ERR_ARG, "bad dtype %d", in_dtype);
  if (targets != KVR_KEYS_ONLY && targets != KVR_KEYS_AND_VALUES) return fail(KVR_ERR_ARG, "bad targets %d", targets);
  if (int rc = check_order(pl.d, rot_order)) return rc;
  if (pl.prec != KVR_PREC_INT4) return fail(KVR_ERR_UNSUPPORTED, "learned store: INT4 pools only");
  Signs s;
  int has;
  if (int rc = make_signs(sign_words, pl.d, s, has)) return rc;
  if (n_tok == 0) return KVR_OK;
  const int mode_v = targets == KVR_KEYS_ONLY ? 0 : (learned_values ? 2 : 1);
  cudaStream_t st = (cudaStream_t)stream;
  kvr_mark_pool_written(st);
  const int rc = kvr_launch_store_learned(k, v, in_dtype, n_tok, slot_mapping, pl, rot_order, mode_v, s, has, t_img,
                                          r_t, flags, st);
  if (rc == KVR_ERR_UNSUPPORTED)
    return fail(rc, "learned store: bf16 rows, d = 128, 16-token cells, power-of-two pages, 16-B aligned only");
  if (rc) return fail(rc, "rotate_quantize_store_learned: launch failed (%d)", rc);
  return check_launch("rotate_quantize_store_learned");
}

void kvr_learned_pack_image(const double* t, uint16_t* img) {
  if (t && img) kvr_pack_learned_image(t, img);
}

int kvr_dequantize_pages(const kvr_pool* pool, const int32_t* block_table, int32_t bt_stride,
                         const int32_t* seq_lens, int32_t batch, int32_t max_len, void* k_out, void* v_out,
                         int32_t out_dtype, void* stream) {
  Pool pl;
  if (int rc = to_pool(pool, pl)) return rc;
  if (batch < 0 || max_len < 0) return fail(KVR_ERR_SHAPE, "bad batch/max_len");
  if (batch == 0 || max_len == 0) return KVR_OK;
  int rc = kvr_launch_dequant_pages(pl, block_table, bt_stride, seq_lens, batch, max_len, k_out, v_out, out_dtype,
                                    (cudaStream_t)stream);
  if (rc) return fail(rc, "dequantize_pages: unsupported out dtype %d", out_dtype);
  return check_launch("dequantize_pages");
}

int kvr_decode_flat_f64(const double* q, const double* k, const double* v, int64_t t, int32_t num_q_heads,
                        int32_t num_kv_heads, int32_t head_dim, double* out, void* stream) {
  if (t < 1 || num_kv_heads < 1 || num_q_heads < 1 || num_q_heads % num_kv_heads || head_dim < 1)
    return fail(KVR_ERR_SHAPE, "decode_flat_f64: bad shape (t=%lld, nq=%d, H=%d, d=%d)", (long long)t, num_q_heads,
                num_kv_heads, head_dim);
  if (!q || !k || !v || !out) return fail(KVR_ERR_ARG, "decode_flat_f64: null pointer");
  if (int rc = kvr_launch_decode_flat_f64(q, k, v, t, num_q_heads, num_kv_heads, head_dim, out, (cudaStream_t)stream))
    return fail(rc, "decode_flat_f64: head_dim %d > 256", head_dim);
  return check_launch("decode_flat_f64");
}

size_t kvr_decode_workspace_bytes(int32_t batch, int32_t num_kv_heads, int32_t num_q_heads, int32_t head_dim,
                                  int32_t num_splits) {
  return kvr_decode_ws_bytes(batch, num_kv_heads, num_q_heads, head_dim, num_splits);
}

int kvr_decode_pick_splits(int32_t batch, int32_t num_kv_heads, int32_t max_seq_len, int32_t page_tokens) {
  return kvr_pick_splits(batch, num_kv_heads, max_seq_len, page_tokens);
}

int kvr_paged_decode(const void* q, int32_t q_dtype, const kvr_pool* pool, const int32_t* block_table,
                     int32_t bt_stride, const int32_t* seq_lens, int32_t batch, int32_t num_q_heads,
                     int32_t max_seq_len, int32_t rot_order, int32_t rotate, int32_t targets,
                     const uint32_t* sign_words, float* out, void* workspace, size_t workspace_bytes,
                     int32_t num_splits, void* stream) {
  Pool pl;
  if (int rc = to_pool(pool, pl)) return rc;
  if (batch < 0 || num_q_heads < 1 || num_q_heads % pl.H != 0)
    return fail(KVR_ERR_SHAPE, "num_q_heads=%d is not a multiple of num_kv_heads=%d", num_q_heads, pl.H);
  if (batch == 0) return KVR_OK;
  if (max_seq_len < 0 || (int64_t)bt_stride * pl.P < max_seq_len)
    return fail(KVR_ERR_SHAPE, "max_seq_len=%d exceeds bt_stride=%d pages of %d tokens", max_seq_len, bt_stride, pl.P);
  if (q_dtype != KVR_F32 && q_dtype != KVR_BF16 && q_dtype != KVR_F16)
    return fail(KVR_ERR_ARG, "q dtype %d unsupported (F32/BF16/F16)", q_dtype);
  if (pl.prec == KVR_PREC_BF16) rotate = 0;  // raw vectors: the query is used as-is (attention.py:67-71)
  if (rotate) {
    if (int rc = check_order(pl.d, rot_order)) return rc;
  } else {
    rot_order = 1;
  }
  Signs s;
  int has;
  if (int rc = make_signs(rotate ? sign_words : nullptr, pl.d, s, has)) return rc;
  const int rot_v = (rotate && targets == KVR_KEYS_AND_VALUES) ? 1 : 0;
  int rc = kvr_launch_decode(q, q_dtype, pl, block_table, bt_stride, seq_lens, batch, num_q_heads, max_seq_len,
                             rot_order, rotate, rot_v, s, has, out, workspace, workspace_bytes, num_splits,
                             (cudaStream_t)stream);
  if (rc == KVR_ERR_ARG) return fail(rc, "decode workspace too small");
  if (rc) return fail(rc, "paged_decode: unsupported geometry (d=%d, P=%d, G=%d)", pl.d, pl.P, num_q_heads / pl.H);
  return check_launch("paged_decode");
}

int kvr_paged_decode_learned(const void* q, int32_t q_dtype, const kvr_pool* pool, const int32_t* block_table,
                             int32_t bt_stride, const int32_t* seq_lens, int32_t batch, int32_t num_q_heads,
                             int32_t max_seq_len, const float* t_pad, int32_t out_mode, int32_t rot_order,
                             const uint32_t* sign_words, float* out, void* workspace, size_t workspace_bytes,
                             int32_t num_splits, void* stream) {
  Pool pl;
  if (int rc = to_pool(pool, pl)) return rc;
  if (batch < 0 || num_q_heads < 1 || num_q_heads % pl.H != 0)
    return fail(KVR_ERR_SHAPE, "num_q_heads=%d is not a multiple of num_kv_heads=%d", num_q_heads, pl.H);
  if (!t_pad || (reinterpret_cast<uintptr_t>(t_pad) & 15)) return fail(KVR_ERR_ARG, "t_pad must be 16-B aligned");
  if (out_mode < 0 || out_mode > 2) return fail(KVR_ERR_ARG, "out_mode=%d (0, 1 or 2)", out_mode);
  if (batch == 0) return KVR_OK;
  if (max_seq_len < 0 || (int64_t)bt_stride * pl.P < max_seq_len)
    return fail(KVR_ERR_SHAPE, "max_seq_len=%d exceeds bt_stride=%d pages of %d tokens", max_seq_len, bt_stride, pl.P);
  if (q_dtype != KVR_F32 && q_dtype != KVR_BF16 && q_dtype != KVR_F16)
    return fail(KVR_ERR_ARG, "q dtype %d unsupported (F32/BF16/F16)", q_dtype);
  const int G = num_q_heads / pl.H;
  if (pl.prec != KVR_PREC_INT4 || pl.d != 128 || pl.T != 16 || (pl.P & (pl.P - 1)) ||
      !(G == 1 || G == 2 || G == 4 || G == 8))
    return fail(KVR_ERR_UNSUPPORTED, "paged_decode_learned: INT4, d = 128, power-of-two pages, G in 1/2/4/8");
  Signs s;
  int has = 0;
  if (out_mode == 1) {
    if (int rc = check_order(pl.d, rot_order)) return rc;
    if (int rc = make_signs(sign_words, pl.d, s, has)) return rc;
  } else {
    rot_order = 1;
    if (int rc = make_signs(nullptr, pl.d, s, has)) return rc;
  }
  const int rc = kvr_launch_decode(q, q_dtype, pl, block_table, bt_stride, seq_lens, batch, num_q_heads, max_seq_len,
                                   128, 0, 0, s, has, out, workspace, workspace_bytes, num_splits, (cudaStream_t)stream,
                                   nullptr, nullptr, 0, nullptr, nullptr, 0, t_pad, out_mode, rot_order);
  if (rc == KVR_ERR_ARG) return fail(rc, "decode workspace too small");
  if (rc) return fail(rc, "paged_decode_learned: unsupported geometry (d=%d, P=%d, G=%d)", pl.d, pl.P, G);
  return check_launch("paged_decode_learned");
}

int kvr_decode_step(const void* q, int32_t q_dtype, const void* new_k, const void* new_v, int32_t kv_dtype,
                    const int64_t* new_slot, const kvr_pool* pool, const int32_t* block_table, int32_t bt_stride,
                    const int32_t* seq_lens, int32_t batch, int32_t num_q_heads, int32_t max_seq_len,
                    int32_t rot_order, int32_t rotate, int32_t targets, const uint32_t* sign_words, float* out,
                    void* workspace, size_t workspace_bytes, int32_t num_splits, uint32_t* flags, void* stream) {
  return decode_step_impl(q, q_dtype, new_k, new_v, kv_dtype, new_slot, pool, block_table, bt_stride, seq_lens, batch,
                          num_q_heads, max_seq_len, rot_order, rotate, targets, sign_words, out, workspace,
                          workspace_bytes, num_splits, flags, stream, 0);
}

}  // extern "C"

static int decode_step_impl(const void* q, int32_t q_dtype, const void* new_k, const void* new_v, int32_t kv_dtype,
                            const int64_t* new_slot, const kvr_pool* pool, const int32_t* block_table,
                            int32_t bt_stride, const int32_t* seq_lens, int32_t batch, int32_t num_q_heads,
                            int32_t max_seq_len, int32_t rot_order, int32_t rotate, int32_t targets,
                            const uint32_t* sign_words, float* out, void* workspace, size_t workspace_bytes,
                            int32_t num_splits, uint32_t* flags, void* stream, int q_host_staged) {
  Pool pl;
  if (int rc = to_pool(pool, pl)) return rc;
  if (batch < 0 || num_q_heads < 1 || num_q_heads % pl.H != 0)
    return fail(KVR_ERR_SHAPE, "num_q_heads=%d is not a multiple of num_kv_heads=%d", num_q_heads, pl.H);
  if (batch == 0) return KVR_OK;
  if (max_seq_len < 0 || (int64_t)bt_stride * pl.P < max_seq_len)
    return fail(KVR_ERR_SHAPE, "max_seq_len=%d exceeds bt_stride=%d pages of %d tokens", max_seq_len, bt_stride, pl.P);
  if (!new_k || !new_v || !new_slot) return fail(KVR_ERR_ARG, "decode_step needs new_k, new_v and new_slot");
  if (kv_dtype < KVR_F64 || kv_dtype > KVR_F16) return fail(KVR_ERR_ARG, "bad kv dtype %d", kv_dtype);
  if (q_dtype != KVR_F32 && q_dtype != KVR_BF16 && q_dtype != KVR_F16)
    return fail(KVR_ERR_ARG, "q dtype %d unsupported (F32/BF16/F16)", q_dtype);
  if (pl.prec == KVR_PREC_BF16) {
    // BF16 pool: write the raw new rows, then a plain decode with the query as-is
    kvr_mark_pool_written((cudaStream_t)stream);
    if (int rc = kvr_launch_store_bf16(new_k, new_v, kv_dtype, batch, new_slot, pl, flags, (cudaStream_t)stream))
      return fail(rc, "decode_step (bf16 pool): store failed (%d)", rc);
    Signs s0;
    int has0;
    make_signs(nullptr, pl.d, s0, has0);
    int rc = kvr_launch_decode(q, q_dtype, pl, block_table, bt_stride, seq_lens, batch, num_q_heads, max_seq_len, 1,
                               0, 0, s0, has0, out, workspace, workspace_bytes, num_splits, (cudaStream_t)stream);
    if (rc == KVR_ERR_ARG) return fail(rc, "decode workspace too small");
    if (rc) return fail(rc, "decode_step (bf16 pool): unsupported geometry (d=%d)", pl.d);
    return check_launch("decode_step");
  }
  if (rotate) {
    if (int rc = check_order(pl.d, rot_order)) return rc;
  } else {
    rot_order = 1;
  }
  Signs s;
  int has;
  if (int rc = make_signs(rotate ? sign_words : nullptr, pl.d, s, has)) return rc;
  const int rot_v = (rotate && targets == KVR_KEYS_AND_VALUES) ? 1 : 0;
  int rc = kvr_launch_decode(q, q_dtype, pl, block_table, bt_stride, seq_lens, batch, num_q_heads, max_seq_len,
                             rot_order, rotate, rot_v, s, has, out, workspace, workspace_bytes, num_splits,
                             (cudaStream_t)stream, new_k, new_v, kv_dtype, new_slot, flags, q_host_staged);
  if (rc == KVR_ERR_ARG) return fail(rc, "decode workspace too small");
  if (rc) return fail(rc, "decode_step: unsupported geometry (needs d=128, page_tokens>=16, G in 1/2/4/8)");
  return check_launch("decode_step");
}
