// radix_sort.cu — host driver of the hand-written radix sort (radix_sort.cuh) used by the CSF
// builder for every sort of nonzeros or nodes.
#include "csf.hpp"
#include "radix_sort.cuh"

namespace sb {

namespace {

// 8-bit digits, 256 threads x 16 pairs per tile, two CTAs per SM (B200 sweep,
// profiles/ab_r02/onesweep_bench.cu: faster than CUB's onesweep on 57-bit keys and on the
// 14-18-bit root re-sorts; 9-bit digits and larger tiles lose).
constexpr int kBits = 8, kThreads = 256;
// pairs per thread: 16 (12 with 8-byte values, so two CTAs still fit in shared memory)
template <typename V>
constexpr int ipt() { return sizeof(V) == 8 ? 12 : 16; }

template <typename K, typename V>
void sort_impl(splatt_ctx* ctx, const K* src_k, const V* src_v, K* out_k, V* out_v,
               K* tmp_k, V* tmp_v, uint64_t n, int begin, int end) {
  constexpr int kIpt = ipt<V>();
  using P = rs::Pass<K, V, kBits, kThreads, kIpt>;
  cudaStream_t st = ctx->stream;
  if (n == 0) return;
  if (n >= (1ull << 31)) fail(SPLATT_ERR_UNSUPPORTED, "radix sort: n >= 2^31");
  const int npass = end > begin ? (end - begin + kBits - 1) / kBits : 0;
  if (npass == 0) {
    if (out_k != src_k) SB_CUDA(cudaMemcpyAsync(out_k, src_k, n * sizeof(K), cudaMemcpyDeviceToDevice, st));
    if (out_v != src_v) SB_CUDA(cudaMemcpyAsync(out_v, src_v, n * sizeof(V), cudaMemcpyDeviceToDevice, st));
    return;
  }
  auto aligned = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  if (!aligned(src_k) || !aligned(src_v) || !aligned(out_k) || !aligned(out_v) ||
      !aligned(tmp_k) || !aligned(tmp_v))
    fail(SPLATT_ERR_CUDA, "internal: radix sort buffers must be 16-byte aligned");
  // Destinations alternate so that the last pass writes `out`; the source is read by pass 0
  // only, so `tmp` may be the source itself when pass 0 writes `out` (odd pass count).
  DevBuf<K> xk;
  DevBuf<V> xv;
  if ((npass % 2 == 0) && (tmp_k == src_k || tmp_v == src_v)) {
    xk.alloc(n, st);
    xv.alloc(n, st);
    tmp_k = xk.p;
    tmp_v = xv.p;
  }
  set_max_dynamic_smem((const void*)rs::downsweep_kernel<K, V, kBits, kThreads, kIpt>, (int)P::kSmem);
  static thread_local int ctas = 0;
  if (!ctas) ctas = rs::downsweep_ctas_per_sm<K, V, kBits, kThreads, kIpt>();
  const uint64_t ntiles = ceil_div(n, P::kTile);
  const uint64_t C = (uint64_t)ctx->num_sms * ctas;
  const uint32_t tpr = (uint32_t)ceil_div(ntiles, C);
  const int nranges = (int)ceil_div(ntiles, tpr);
  DevBuf<uint32_t> counts((size_t)nranges * P::B, st);
  const K* ik = src_k;
  const V* iv = src_v;
  for (int p = 0; p < npass; ++p) {
    const bool to_out = ((npass - 1 - p) % 2) == 0;
    K* ok = to_out ? out_k : tmp_k;
    V* ov = to_out ? out_v : tmp_v;
    const int shift = begin + p * kBits;
    const uint32_t mask = (1u << std::min(kBits, end - shift)) - 1u;
    rs::upsweep_kernel<K, kBits><<<nranges, 512, 0, st>>>(ik, (uint32_t)n, shift, mask,
                                                          tpr * (uint32_t)P::kTile, counts.p);
    SB_CHECK_LAUNCH(ctx);
    rs::scan_kernel<kBits><<<1, 1024, 0, st>>>(counts.p, nranges);
    SB_CHECK_LAUNCH(ctx);
    rs::downsweep_kernel<K, V, kBits, kThreads, kIpt><<<nranges, kThreads, P::kSmem, st>>>(
        ik, ok, iv, ov, (uint32_t)n, shift, mask, tpr, counts.p);
    SB_CHECK_LAUNCH(ctx);
    ik = ok;
    iv = ov;
  }
}

}  // namespace

void radix_sort_pairs(splatt_ctx* ctx, const uint64_t* src_k, const uint32_t* src_v,
                      uint64_t* out_k, uint32_t* out_v, uint64_t* tmp_k, uint32_t* tmp_v,
                      uint64_t n, int begin, int end) {
  sort_impl<uint64_t, uint32_t>(ctx, src_k, src_v, out_k, out_v, tmp_k, tmp_v, n, begin, end);
}

void radix_sort_pairs(splatt_ctx* ctx, const uint64_t* src_k, const uint64_t* src_v,
                      uint64_t* out_k, uint64_t* out_v, uint64_t* tmp_k, uint64_t* tmp_v,
                      uint64_t n, int begin, int end) {
  sort_impl<uint64_t, uint64_t>(ctx, src_k, src_v, out_k, out_v, tmp_k, tmp_v, n, begin, end);
}

void radix_sort_pairs(splatt_ctx* ctx, const uint32_t* src_k, const uint32_t* src_v,
                      uint32_t* out_k, uint32_t* out_v, uint32_t* tmp_k, uint32_t* tmp_v,
                      uint64_t n, int begin, int end) {
  sort_impl<uint32_t, uint32_t>(ctx, src_k, src_v, out_k, out_v, tmp_k, tmp_v, n, begin, end);
}

}  // namespace sb
