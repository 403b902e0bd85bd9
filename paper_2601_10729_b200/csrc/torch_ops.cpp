// torch.library registration of the data-path ops (the
// `orbit::` extension ops) - a thin layer over the same C ABI
// (include/orbitflow_b200.h) that the ctypes binding calls, so both bindings
// run the identical sm_100a kernels.  Registering them with the dispatcher
// makes them visible to torch.ops, to CUDA-graph capture through torch.ops and
// to torch.compile (fake kernels live in ops.py).  CUDA tensors only: there is
// no CPU kernel, a CPU tensor raises (the north star forbids a CPU fallback).
//
//   orbit::decode_attention  K1  (priced by kvsim/core.py:257-261)
//   orbit::kv_append         K3  (kvsim/core.py:95-102, engine.py:389-392)
//   orbit::kv_prefill        K5  (engine.py:495-503)
//   orbit::decode_step       K3+K2+K1 of one step (engine.py:715-734)
//   orbit::migrate           K4  (apply_plan, engine.py:213-248)
#include <ATen/ATen.h>
#include <ATen/cuda/CUDAContext.h>
#include <torch/library.h>

#include <cmath>
#include <string>

#include "orbitflow_b200.h"

namespace {

void check_rc(int rc, const char* what) {
  TORCH_CHECK(rc == 0, what, " failed (rc=", rc, "): ", ofb_last_error());
}

void* cur_stream(const at::Tensor& t) {
  return reinterpret_cast<void*>(at::cuda::getCurrentCUDAStream(t.device().index()).stream());
}

void need_cuda(const at::Tensor& t, const char* name) {
  TORCH_CHECK(t.is_cuda(), "orbit: ", name, " must be a CUDA tensor (no CPU fallback)");
}

// out = softmax(scale q K^T) V over the paged KV of one layer.
at::Tensor decode_attention_out(const at::Tensor& q, const at::Tensor& kv_pool,
                                const at::Tensor& block_tables, const at::Tensor& seq_lens,
                                int64_t max_seq_len, double scale, const at::Tensor& ws,
                                at::Tensor& out) {
  need_cuda(q, "q");
  need_cuda(kv_pool, "kv_pool");
  need_cuda(block_tables, "block_tables");
  need_cuda(seq_lens, "seq_lens");
  need_cuda(ws, "ws");
  need_cuda(out, "out");
  TORCH_CHECK(q.scalar_type() == at::kBFloat16 && kv_pool.scalar_type() == at::kBFloat16,
              "orbit::decode_attention: q and kv_pool must be bf16");
  TORCH_CHECK(block_tables.scalar_type() == at::kInt && seq_lens.scalar_type() == at::kInt,
              "orbit::decode_attention: block_tables and seq_lens must be int32");
  TORCH_CHECK(q.dim() == 3 && q.size(2) == 128, "orbit::decode_attention: q must be [B, Hq, 128]");
  TORCH_CHECK(kv_pool.dim() == 5 && kv_pool.size(2) == 2 && kv_pool.size(3) == 16 &&
                  kv_pool.size(4) == 128,
              "orbit::decode_attention: kv_pool must be [blocks, Hkv, 2, 16, 128]");
  TORCH_CHECK(q.is_contiguous() && block_tables.is_contiguous() && out.is_contiguous() &&
                  kv_pool.is_contiguous(),
              "orbit::decode_attention: contiguous tensors required");
  TORCH_CHECK(out.sizes() == q.sizes() && out.scalar_type() == q.scalar_type(),
              "orbit::decode_attention: out must match q");
  const int32_t batch = static_cast<int32_t>(q.size(0));
  const int32_t hq = static_cast<int32_t>(q.size(1));
  const int32_t hkv = static_cast<int32_t>(kv_pool.size(1));
  const int64_t need = ofb_attention_workspace_bytes(batch, hq, hkv, static_cast<int32_t>(max_seq_len));
  TORCH_CHECK(ws.numel() * ws.element_size() >= need,
              "orbit::decode_attention: workspace too small (", need, " bytes needed)");
  check_rc(ofb_decode_attention(q.data_ptr(), out.data_ptr(), kv_pool.data_ptr(), kv_pool.size(0),
                                block_tables.data_ptr<int32_t>(),
                                static_cast<int32_t>(block_tables.size(-1)),
                                seq_lens.data_ptr<int32_t>(), ws.data_ptr(),
                                ws.numel() * ws.element_size(), batch, hq, hkv, 128,
                                static_cast<int32_t>(max_seq_len), static_cast<float>(scale),
                                cur_stream(q)),
           "orbit::decode_attention");
  return out;
}

at::Tensor decode_attention(const at::Tensor& q, const at::Tensor& kv_pool,
                            const at::Tensor& block_tables, const at::Tensor& seq_lens,
                            int64_t max_seq_len, double scale, const at::Tensor& ws) {
  at::Tensor out = at::empty_like(q);
  return decode_attention_out(q, kv_pool, block_tables, seq_lens, max_seq_len, scale, ws, out);
}

// k_new/v_new: bf16 [L, B, Hkv, 128]; block_tables int32 [L, B, max_blocks];
// host_slabs: int64 [L, B] mapped host slab bases (0 = none) or None.
void kv_append(const at::Tensor& k_new, const at::Tensor& v_new, at::Tensor& kv_pool,
               const at::Tensor& block_tables, const at::Tensor& positions,
               const std::optional<at::Tensor>& host_slabs) {
  need_cuda(k_new, "k_new");
  need_cuda(v_new, "v_new");
  need_cuda(kv_pool, "kv_pool");
  need_cuda(block_tables, "block_tables");
  need_cuda(positions, "positions");
  TORCH_CHECK(k_new.dim() == 4 && k_new.sizes() == v_new.sizes() && k_new.size(3) == 128,
              "orbit::kv_append: k_new/v_new must be [L, B, Hkv, 128]");
  TORCH_CHECK(k_new.is_contiguous() && v_new.is_contiguous() && block_tables.is_contiguous(),
              "orbit::kv_append: contiguous tensors required");
  TORCH_CHECK(block_tables.dim() == 3 && block_tables.scalar_type() == at::kInt &&
                  positions.scalar_type() == at::kInt,
              "orbit::kv_append: int32 block_tables [L, B, max_blocks] and positions [B]");
  const uint64_t* hs = nullptr;
  if (host_slabs.has_value()) {
    need_cuda(*host_slabs, "host_slabs");
    TORCH_CHECK(host_slabs->scalar_type() == at::kLong && host_slabs->is_contiguous(),
                "orbit::kv_append: host_slabs must be contiguous int64 [L, B]");
    hs = reinterpret_cast<const uint64_t*>(host_slabs->data_ptr<int64_t>());
  }
  check_rc(ofb_kv_append(k_new.data_ptr(), v_new.data_ptr(), kv_pool.data_ptr(),
                         block_tables.data_ptr<int32_t>(),
                         static_cast<int32_t>(block_tables.size(-1)), positions.data_ptr<int32_t>(),
                         hs, static_cast<int32_t>(k_new.size(0)), static_cast<int32_t>(k_new.size(1)),
                         static_cast<int32_t>(k_new.size(2)), 128, cur_stream(k_new)),
           "orbit::kv_append");
}

// k/v: bf16 [L, P, Hkv, 128] prompt KV; dst: int64 [L] slab base addresses.
void kv_prefill(const at::Tensor& k, const at::Tensor& v, const at::Tensor& dst) {
  need_cuda(k, "k");
  need_cuda(v, "v");
  need_cuda(dst, "dst");
  TORCH_CHECK(k.dim() == 4 && k.sizes() == v.sizes() && k.is_contiguous() && v.is_contiguous(),
              "orbit::kv_prefill: k/v must be contiguous [L, P, Hkv, 128]");
  TORCH_CHECK(dst.scalar_type() == at::kLong && dst.numel() == k.size(0),
              "orbit::kv_prefill: dst must be int64 [L]");
  check_rc(ofb_kv_prefill(k.data_ptr(), v.data_ptr(),
                          reinterpret_cast<const uint64_t*>(dst.data_ptr<int64_t>()),
                          static_cast<int32_t>(k.size(0)), static_cast<int32_t>(k.size(1)),
                          static_cast<int32_t>(k.size(2)), 128, cur_stream(k)),
           "orbit::kv_prefill");
}

// One whole decode step through the native runtime.  `runtime` is the
// ofb_runtime handle and `desc` the address of a filled ofb_step_desc (its
// device tensors are the ones the caller passes in `out`, which the step
// writes); both come from executor.B200Executor, which owns them.
void decode_step(int64_t runtime, int64_t desc, at::Tensor& out) {
  need_cuda(out, "out");
  auto* d = reinterpret_cast<const ofb_step_desc*>(desc);
  TORCH_CHECK(runtime != 0 && d != nullptr, "orbit::decode_step: null runtime or descriptor");
  TORCH_CHECK(d->out == out.data_ptr(), "orbit::decode_step: out is not the descriptor's output");
  check_rc(ofb_runtime_decode_step(reinterpret_cast<ofb_runtime*>(runtime), d, cur_stream(out)),
           "orbit::decode_step");
}

// Whole-layer migrations (K4): n copies dst[i] <- src[i] of bytes[i],
// kinds[i] 0 = H2D restore, 1 = D2H eviction, 2 = D2D.  Arrays are host int64/int32.
void migrate(int64_t runtime, const at::Tensor& dst, const at::Tensor& src,
             const at::Tensor& bytes, const at::Tensor& kinds, bool record_timing,
             const at::Tensor& stream_of) {
  TORCH_CHECK(!dst.is_cuda() && !src.is_cuda() && !bytes.is_cuda() && !kinds.is_cuda(),
              "orbit::migrate: the transfer list lives in host tensors");
  TORCH_CHECK(dst.scalar_type() == at::kLong && src.scalar_type() == at::kLong &&
                  bytes.scalar_type() == at::kLong && kinds.scalar_type() == at::kInt,
              "orbit::migrate: int64 dst/src/bytes, int32 kinds");
  const int64_t n = dst.numel();
  TORCH_CHECK(src.numel() == n && bytes.numel() == n && kinds.numel() == n,
              "orbit::migrate: ragged transfer list");
  need_cuda(stream_of, "stream_of");
  check_rc(ofb_runtime_migrate(reinterpret_cast<ofb_runtime*>(runtime), static_cast<int32_t>(n),
                               reinterpret_cast<const uint64_t*>(dst.data_ptr<int64_t>()),
                               reinterpret_cast<const uint64_t*>(src.data_ptr<int64_t>()),
                               bytes.data_ptr<int64_t>(), kinds.data_ptr<int32_t>(),
                               record_timing ? 1 : 0, cur_stream(stream_of)),
           "orbit::migrate");
}

}  // namespace

TORCH_LIBRARY(orbit, m) {
  m.def("decode_attention(Tensor q, Tensor kv_pool, Tensor block_tables, Tensor seq_lens, "
        "int max_seq_len, float scale, Tensor ws) -> Tensor");
  m.def("decode_attention.out(Tensor q, Tensor kv_pool, Tensor block_tables, Tensor seq_lens, "
        "int max_seq_len, float scale, Tensor ws, *, Tensor(a!) out) -> Tensor(a!)");
  m.def("kv_append(Tensor k_new, Tensor v_new, Tensor(a!) kv_pool, Tensor block_tables, "
        "Tensor positions, Tensor? host_slabs) -> ()");
  m.def("kv_prefill(Tensor k, Tensor v, Tensor dst) -> ()");
  m.def("decode_step(int runtime, int desc, Tensor(a!) out) -> ()");
  m.def("migrate(int runtime, Tensor dst, Tensor src, Tensor bytes, Tensor kinds, "
        "bool record_timing, Tensor stream_of) -> ()");
}

TORCH_LIBRARY_IMPL(orbit, CUDA, m) {
  m.impl("decode_attention", &decode_attention);
  m.impl("decode_attention.out", &decode_attention_out);
  m.impl("kv_append", &kv_append);
  m.impl("kv_prefill", &kv_prefill);
  m.impl("decode_step", &decode_step);
  m.impl("migrate", &migrate);
}
