/*
 * oracle/kvd_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct CPU implementation of what KVDirect's
 * pull path computes (arXiv 2501.14743, §4.1 "KVDirect
 * Communication Design", and §4.3 pull mode).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * constant or helper with the CUDA path under paper_2501_14743_b200/: the
 * two are independent by construction.
 *
 * What the method computes (plain definition; SURVEY.md §8 row c):
 *   for every i < n, l < NL, kv < 2, t < L(block_size), h < H, d < D:
 *     T_l[dst_ids[i]][kv][t][h][d] = S_l[src_ids[i]][kv][t][h][d]
 *   and every other destination byte keeps its value.
 * Each element's byte address is the paper's dot product of the index
 * with the tensor's stride vector times the element size:
 *   offset(b, kv, t, h, d) = e * (b*s_B + kv*s_KV + t*s_L + h*s_H + d*s_D).
 * No span arithmetic, no runs, no memcpy of spans: every element is
 * addressed and copied on its own, byte by byte.
 *
 * Strides are given in ELEMENTS in the paper's Dims order (B, KV, L, H, D),
 * exactly like Fig. 5.  An all-zero stride vector means the
 * default layout of Fig. 5: K tensors of all blocks first, then the V
 * tensors (stride_KV = B * L*H*D, stride_B = L*H*D, stride_L = H*D,
 * stride_H = D, stride_D = 1), which is the paper's own example layout.
 *
 * Validation (readings R9, R12): a source or destination block id
 * outside [0, num_blocks) -> ORACLE_ERANGE; a destination id that appears
 * twice -> ORACLE_EINVAL (two different sources would race for one block).
 * On error nothing is written.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL (-1)
#define ORACLE_ERANGE (-2)

/* Dims order of Fig. 5: B, KV, L, H, D. */
enum { DIM_B = 0, DIM_KV = 1, DIM_L = 2, DIM_H = 3, DIM_D = 4 };

/* Fig. 5's stride pattern written out for a cache of the given shape. */
void oracle_default_strides(uint32_t num_blocks, uint32_t block_size,
                            uint32_t num_heads, uint32_t head_dim,
                            int64_t stride_out[5]) {
  int64_t sub = (int64_t)block_size * num_heads * head_dim; /* (L,H,D) sub-tensor */
  stride_out[DIM_B] = sub;
  stride_out[DIM_KV] = (int64_t)num_blocks * sub;
  stride_out[DIM_L] = (int64_t)num_heads * head_dim;
  stride_out[DIM_H] = head_dim;
  stride_out[DIM_D] = 1;
}

/* "perform a dot-product between the index and the stride",
 * then multiply by the element size. */
int64_t oracle_element_offset(const int64_t stride[5], const int64_t index[5],
                              uint32_t elem_bytes) {
  int64_t dot = 0;
  for (int k = 0; k < 5; ++k) dot += index[k] * stride[k];
  return dot * (int64_t)elem_bytes;
}

static void resolve_strides(const int64_t in[5], uint32_t num_blocks,
                            uint32_t block_size, uint32_t num_heads,
                            uint32_t head_dim, int64_t out[5]) {
  int all_zero = 1;
  for (int k = 0; k < 5; ++k)
    if (in[k] != 0) all_zero = 0;
  if (all_zero)
    oracle_default_strides(num_blocks, block_size, num_heads, head_dim, out);
  else
    for (int k = 0; k < 5; ++k) out[k] = in[k];
}

static int validate(const int32_t* src_ids, const int32_t* dst_ids, uint32_t n,
                    uint32_t src_num_blocks, uint32_t dst_num_blocks) {
  for (uint32_t i = 0; i < n; ++i) {
    if (src_ids[i] < 0 || (uint32_t)src_ids[i] >= src_num_blocks) return ORACLE_ERANGE;
    if (dst_ids[i] < 0 || (uint32_t)dst_ids[i] >= dst_num_blocks) return ORACLE_ERANGE;
  }
  /* duplicate destination ids: plain O(n^2) pairwise comparison */
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = i + 1; j < n; ++j)
      if (dst_ids[i] == dst_ids[j]) return ORACLE_EINVAL;
  return ORACLE_OK;
}

static void copy_element(uint8_t* dst, const uint8_t* src, uint32_t elem_bytes) {
  for (uint32_t k = 0; k < elem_bytes; ++k) dst[k] = src[k];
}

/*
 * Block-ordered loop: for i (request block), l (layer), kv, t, h, d.
 * src_layers[l] / dst_layers[l] are the base addresses of layer l's cache
 * tensor on each side ("Address" of P:L299; vLLM keeps one tensor per layer).
 */
int oracle_pull_blockwise(const uint8_t* const* src_layers, const int64_t src_stride_in[5],
                          uint32_t src_num_blocks, uint8_t* const* dst_layers,
                          const int64_t dst_stride_in[5], uint32_t dst_num_blocks,
                          uint32_t num_layers, uint32_t num_heads, uint32_t head_dim,
                          uint32_t block_size, uint32_t elem_bytes, const int32_t* src_ids,
                          const int32_t* dst_ids, uint32_t n) {
  int rc = validate(src_ids, dst_ids, n, src_num_blocks, dst_num_blocks);
  if (rc != ORACLE_OK) return rc;
  int64_t ss[5], ds[5];
  resolve_strides(src_stride_in, src_num_blocks, block_size, num_heads, head_dim, ss);
  resolve_strides(dst_stride_in, dst_num_blocks, block_size, num_heads, head_dim, ds);
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t l = 0; l < num_layers; ++l)
      for (int64_t kv = 0; kv < 2; ++kv)
        for (int64_t t = 0; t < block_size; ++t)
          for (int64_t h = 0; h < num_heads; ++h)
            for (int64_t d = 0; d < head_dim; ++d) {
              int64_t si[5] = {src_ids[i], kv, t, h, d};
              int64_t di[5] = {dst_ids[i], kv, t, h, d};
              copy_element(dst_layers[l] + oracle_element_offset(ds, di, elem_bytes),
                           src_layers[l] + oracle_element_offset(ss, si, elem_bytes),
                           elem_bytes);
            }
  return ORACLE_OK;
}

/*
 * Token brute force (SURVEY.md §8 row c, second loop order): walk the
 * request token by token, q < n*block_size, block i = q / L, slot t = q % L.
 * Must produce byte-identical results to the block-ordered loop.
 */
int oracle_pull_tokenwise(const uint8_t* const* src_layers, const int64_t src_stride_in[5],
                          uint32_t src_num_blocks, uint8_t* const* dst_layers,
                          const int64_t dst_stride_in[5], uint32_t dst_num_blocks,
                          uint32_t num_layers, uint32_t num_heads, uint32_t head_dim,
                          uint32_t block_size, uint32_t elem_bytes, const int32_t* src_ids,
                          const int32_t* dst_ids, uint32_t n) {
  int rc = validate(src_ids, dst_ids, n, src_num_blocks, dst_num_blocks);
  if (rc != ORACLE_OK) return rc;
  int64_t ss[5], ds[5];
  resolve_strides(src_stride_in, src_num_blocks, block_size, num_heads, head_dim, ss);
  resolve_strides(dst_stride_in, dst_num_blocks, block_size, num_heads, head_dim, ds);
  uint64_t tokens = (uint64_t)n * block_size;
  for (uint64_t q = 0; q < tokens; ++q) {
    uint64_t i = q / block_size;
    int64_t t = (int64_t)(q % block_size);
    for (uint32_t l = 0; l < num_layers; ++l)
      for (int64_t h = 0; h < num_heads; ++h)
        for (int64_t kv = 0; kv < 2; ++kv)
          for (int64_t d = 0; d < head_dim; ++d) {
            int64_t si[5] = {src_ids[i], kv, t, h, d};
            int64_t di[5] = {dst_ids[i], kv, t, h, d};
            copy_element(dst_layers[l] + oracle_element_offset(ds, di, elem_bytes),
                         src_layers[l] + oracle_element_offset(ss, si, elem_bytes),
                         elem_bytes);
          }
  }
  return ORACLE_OK;
}

/*
 * TP-resharding pull (not in the paper, which keeps the
 * prefill and decode TP degrees equal).  The prefill shard holds src_heads
 * KV heads, the decode shard dst_heads >= src_heads; the prefill shard's
 * heads land at decode heads [head_offset, head_offset + src_heads):
 *   T_l[dst_ids[i]][kv][t][head_offset + h][d] = S_l[src_ids[i]][kv][t][h][d]
 * for h < src_heads, every other destination byte unchanged.  E.g. prefill
 * TP=8 -> decode TP=4: decode shard j pulls prefill shard 2j at offset 0 and
 * shard 2j+1 at offset src_heads.  Same element loop, same validation.
 */
int oracle_pull_heads(const uint8_t* const* src_layers, const int64_t src_stride_in[5],
                      uint32_t src_num_blocks, uint32_t src_heads, uint8_t* const* dst_layers,
                      const int64_t dst_stride_in[5], uint32_t dst_num_blocks,
                      uint32_t dst_heads, uint32_t head_offset, uint32_t num_layers,
                      uint32_t head_dim, uint32_t block_size, uint32_t elem_bytes,
                      const int32_t* src_ids, const int32_t* dst_ids, uint32_t n) {
  if (head_offset + src_heads > dst_heads) return ORACLE_EINVAL;
  int rc = validate(src_ids, dst_ids, n, src_num_blocks, dst_num_blocks);
  if (rc != ORACLE_OK) return rc;
  int64_t ss[5], ds[5];
  resolve_strides(src_stride_in, src_num_blocks, block_size, src_heads, head_dim, ss);
  resolve_strides(dst_stride_in, dst_num_blocks, block_size, dst_heads, head_dim, ds);
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t l = 0; l < num_layers; ++l)
      for (int64_t kv = 0; kv < 2; ++kv)
        for (int64_t t = 0; t < block_size; ++t)
          for (int64_t h = 0; h < src_heads; ++h)
            for (int64_t d = 0; d < head_dim; ++d) {
              int64_t si[5] = {src_ids[i], kv, t, h, d};
              int64_t di[5] = {dst_ids[i], kv, t, h + head_offset, d};
              copy_element(dst_layers[l] + oracle_element_offset(ds, di, elem_bytes),
                           src_layers[l] + oracle_element_offset(ss, si, elem_bytes),
                           elem_bytes);
            }
  return ORACLE_OK;
}

/*
 * Single-element read used for sampled checks at full size: the byte
 * address of element (b, kv, t, h, d) of one layer, so a test can compute
 * what one output element must be without materialising the whole cache.
 */
int64_t oracle_layer_element_offset(const int64_t stride_in[5], uint32_t num_blocks,
                                    uint32_t block_size, uint32_t num_heads,
                                    uint32_t head_dim, uint32_t elem_bytes, int64_t b,
                                    int64_t kv, int64_t t, int64_t h, int64_t d) {
  int64_t s[5];
  resolve_strides(stride_in, num_blocks, block_size, num_heads, head_dim, s);
  int64_t idx[5] = {b, kv, t, h, d};
  return oracle_element_offset(s, idx, elem_bytes);
}
