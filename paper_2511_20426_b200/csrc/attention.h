// Host interface of the tcgen05 flash attention (attention.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bcb200.h"

namespace bc {

// Kernel parameter block (by value).
struct AttnParams {
  int q_tokens;    // query rows per entry
  int kv_tokens;   // keys per slot (per matrix)
  int heads;
  int mat_base;    // matrix index of slot 0's K for this layer
  int mat_stride;  // matrices between consecutive slots
  int v_offset;    // matrices from a slot's K to its V
  float scale;     // softmax scale (1/sqrt(head_dim))
  void* out;       // bf16 [n_entries*q_tokens][heads*128]
  unsigned long long* trace;  // diagnostic timeline (BC_ATTN_TRACE builds)
  int n_vis[BC_MAX_ENTRIES];
  int vis_slot[BC_MAX_ENTRIES][BC_MAX_VIS];
  // multi-GPU: before the first tile of visible slot v, wait until
  // flags[(flag_base + slot) * n_ranks + r] >= need >> 8 for every producer
  // rank r in the mask need & 0xff (need = 0: no wait; peers publish)
  const uint32_t* flags;
  int flag_base;
  int n_ranks;
  uint32_t need[BC_MAX_ENTRIES][BC_MAX_VIS];
  // query rows of entry e handled by this launch: tokens [q_lo, q_hi), token
  // q_lo at row q_row of the q / out buffers (row-sharded multi-GPU steps
  // run a slice of the batch's rows; by default the whole entry)
  int q_lo[BC_MAX_ENTRIES], q_hi[BC_MAX_ENTRIES], q_row[BC_MAX_ENTRIES];
};

// Work list of the balanced persistent kernel (by value, next to
// AttnParams: the two stay under the 32 KB kernel-parameter limit).  CTA c
// runs items [start[c], start[c+1]).  Item words:
//   e | head << 8 | tile << 16 [| kItemPair]: query tile `tile` (128 rows,
//     counted from the entry's q_lo) of entry e, and with kItemPair also
//     tile + 1 as the ping-pong partner;
//   e | head << 8 | e2 << 16 | kItemCross: the last query tiles of entries e
//     and e2, which attend to identical visible lists (bidirectional mode),
//     as one ping-pong pair.
constexpr uint32_t kItemPair = 0x80000000u;
constexpr uint32_t kItemCross = 0x40000000u;
constexpr int kSchedCtas = 256;
constexpr int kSchedItems = 6144;
struct AttnSched {
  uint16_t start[kSchedCtas + 1];
  uint32_t items[kSchedItems];
};

struct AttnArgs {
  const void* q;        // bf16 [n_entries*q_tokens][heads*128]
  const void* kv_base;  // bf16 matrices [n_mats][kv_tokens][heads*128]
  int n_mats;
  int n_entries, q_tokens, kv_tokens, heads, head_dim;
  int mat_base, mat_stride, v_offset;
  float scale;
  void* out;
  int n_vis[BC_MAX_ENTRIES];
  int vis_slot[BC_MAX_ENTRIES][BC_MAX_VIS];
  const uint32_t* flags;
  int flag_base;
  int n_ranks;
  uint32_t need[BC_MAX_ENTRIES][BC_MAX_VIS];
  // ranged = 0: every entry's q_tokens rows, entry e at row e * q_tokens;
  // ranged = 1: q_lo / q_hi / q_row as in AttnParams, q / out have q_rows rows
  int ranged, q_rows;
  int q_lo[BC_MAX_ENTRIES], q_hi[BC_MAX_ENTRIES], q_row[BC_MAX_ENTRIES];
  // 1: balanced persistent kernel (work list of query-tile items per CTA).
  // Used by single-GPU and multi-GPU steps alike; with peer flags each item
  // waits (bounded, %globaltimer) before its first key tile of a visible
  // slot until every producer rank of that slot published the slot's epoch
  int balance;
};

int attention_run(const AttnArgs& a, cudaStream_t st);

}  // namespace bc
