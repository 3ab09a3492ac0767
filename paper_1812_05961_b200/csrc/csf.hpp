// csf.hpp — device-resident compressed sparse fiber tensors.
#pragma once
#include <memory>

#include "ctx.hpp"

namespace sb {

// Privatised hot output rows per lane group in the INTERNAL / LEAF MTTKRP.
#ifndef SB_HOT_ROWS
#define SB_HOT_ROWS 8
#endif
constexpr int kHotRows = SB_HOT_ROWS;

// Per-tree plan of the second-generation ROOT MTTKRP (root2.cu / root2.cuh): per-leaf
// records {leaf code | d << 29, closing fiber's code, value}, coded ids of levels 1..N-3 and
// the K (level, id) rows held in shared memory.  Built for one padded rank `ld` (K depends
// on the row size).
struct RootPlan {
  int ld = 0;
  uint32_t K = 0;
  DevBuf<uint4> rec;
  DevBuf<uint32_t> cid[SPLATT_MAX_NMODES];
  DevBuf<uint32_t> hot;
  // while the builder forms the plan (root_plan_begin .. root_plan_end): (level, id) -> slot
  DevBuf<uint32_t> slotmap;
  uint64_t off[SPLATT_MAX_NMODES + 1] = {0};
  bool ready = false;
};

// What the builder's level-flag kernel writes per leaf for a plan under construction.
struct RootPlanRecOut {
  uint4* rec = nullptr;        // nullptr: no plan
  const uint32_t* slotmap = nullptr;
  uint64_t off_leaf = 0, off_fiber = 0;  // slotmap offsets of levels N-1 and N-2
  uint32_t ldb = 0;                      // row bytes (ld * 8)
  const double* vals = nullptr;          // the tree's sorted values
};

// One CSF tree.  Level l < N-1: ids[l] (nodes[l]) and ptr[l] (nodes[l]+1, offsets into
// level l+1); leaf level N-1: ids[N-1] (nnz) and vals (nnz).  perm[l] = mode at level l.
struct DevCsf {
  int N = 0;
  uint64_t nnz = 0;
  int perm[SPLATT_MAX_NMODES] = {0};
  uint64_t nodes[SPLATT_MAX_NMODES] = {0};
  DevBuf<uint32_t> ids[SPLATT_MAX_NMODES];
  DevBuf<uint32_t> ptr[SPLATT_MAX_NMODES];
  DevBuf<double> vals;
  // MTTKRP work table (built on first use for a chunk size): per chunk of `tab_chunk`
  // leaves, the node index at every internal level containing the chunk's first leaf
  // plus a flag word (bit 0: the root slice started before the chunk).
  int tab_chunk = 0;
  uint64_t nchunks = 0;
  DevBuf<uint32_t> tab;
  DevBuf<double> seam;  // MTTKRP scratch: one row per chunk (chunk-seam slices)
  DevBuf<double> tail;  // deterministic mode: the open slice's row at each chunk end
  DevBuf<uint32_t> seamrows;  // deterministic mode: head / tail output rows per chunk
  DevBuf<unsigned> work;      // MTTKRP: dynamic chunk counter
  unsigned work_base = 0;     // its value at the next launch's start
  bool work_seq = false;      // inside a launch sequence (cpd_als): no per-launch zeroing
  uint64_t dims[SPLATT_MAX_NMODES] = {0};  // length of the mode at each level
  // Non-root MTTKRP: the kHotRows (8) most frequent ids of each level (~0u = unused), computed on
  // first use of that level as an output level.
  uint32_t hot[SPLATT_MAX_NMODES][kHotRows];
  // ROOT gathers (level 0): -1 not yet timed (L1::no_allocate), 0 L1::no_allocate, 1
  // L1-allocating.  cpd_als times both on its first two iterations and keeps the faster
  // (DESIGN.md §4.2); the choice changes no arithmetic.
  int l1a = -1;
  // Some mode runs an INTERNAL/LEAF traversal over this tree (policies ONE/TWO): its chunk
  // table uses the non-root kernels' best chunk length (mttkrp_chunk_leaves).
  bool nonroot = false;
  bool hot_ready[SPLATT_MAX_NMODES] = {false};
  // Leaf-mode tiling for the ROOT MTTKRP: when the leaf factor does
  // not fit in L2, the same tree split by leaf-id range into tiles (each a tree with the same
  // level order holding the nonzeros whose leaf id falls in its range), run one after another.
  std::vector<std::unique_ptr<DevCsf>> tiles;
  uint64_t tile_rows = 0;  // leaf ids per tile (0 = not tiled)
  // Allocator the tree was built from (nullptr: the stream-ordered pool).  Members built
  // lazily (chunk table, seam rows, tiles) come from the same one, so they live as long as
  // the tree: a call-arena tree dies with its call, a splatt_csf_build tree with its handle.
  Arena* arena = nullptr;
  std::unique_ptr<RootPlan> plan;  // ROOT kernel v2 (built on first use, mttkrp_prepare)
};

// Split c by leaf id into T tiles of ceil(I_leaf / T) ids (tiles empty of nonzeros skipped).
void tile_tree(splatt_ctx* ctx, DevCsf& c, int T);

// perm: root first, then the other modes by ascending length, ties to the lower id
// (SPEC.md:131).
void csf_perm(int N, const uint64_t* dims, int root, int* perm);

// CSF allocation policy (PAPER.md:469-470 lock vs no-lock): number of
// CSFs, their roots, and for every mode the CSF and level its MTTKRP runs on.
//   ALL: CSF_n rooted at n, every mode at level 0 (ROOT kernel).
//   ONE: one CSF rooted at the shortest mode (ties -> lower id), the rest by ascending
//        length below it; mode at level l -> level-l kernel (INTERNAL / LEAF).
//   TWO: ONE's CSF plus one rooted at the longest mode (last in ascending-length order);
//        both roots -> ROOT on their CSF, the rest -> their level in the first CSF.
void csf_policy(int N, const uint64_t* dims, int policy, int* ncsf, int* roots, int* mode_csf,
                int* mode_level);

// Build CSF rooted at `root` from a device COO (ind[m], vals; nnz entries).
void build_csf(splatt_ctx* ctx, const uint32_t* const* d_ind, const double* d_vals, uint64_t nnz,
               int N, const uint64_t* dims, int root, DevCsf& out);

// Build the trees rooted at roots[0..ntrees) (distinct modes) from one device COO: one full
// sort in the ascending-length mode order, every other tree by a short stable re-sort of
// that order on its root coordinate (csf.cu).  Results are identical to build_csf per root.
void build_csf_set(splatt_ctx* ctx, const uint32_t* const* d_ind, const double* d_vals,
                   uint64_t nnz, int N, const uint64_t* dims, const int* roots, int ntrees,
                   DevCsf* const* outs);

// Second-generation ROOT plan of tree `out` for padded rank `ld`, formed by the builder
// (root2.cu): root_plan_begin (before the level flags; returns false if root2 does not apply)
// selects the hot rows from a sample of the level-order sorted coordinates and fills `ro`,
// with which the flag kernel writes every leaf's record; root_plan_end (after the level
// scatter) writes the coded node-id arrays from the tree's ids.  Both from the current arena.
bool root_plan_begin(splatt_ctx* ctx, DevCsf& out, const uint32_t* const* coord,
                     const double* vals, int ld, RootPlanRecOut* ro);
void root_plan_end(splatt_ctx* ctx, DevCsf& out);

// Stable LSD radix sort (radix_sort.cu) of the pairs (src_k[i], src_v[i]) by key bits
// [begin, end) into (out_k, out_v); (tmp_k, tmp_v) is scratch of n pairs and may be the
// source itself (the source is read by the first pass only).  out and src must not alias.
// Every buffer 16-byte aligned; n < 2^31.
void radix_sort_pairs(splatt_ctx* ctx, const uint64_t* src_k, const uint32_t* src_v,
                      uint64_t* out_k, uint32_t* out_v, uint64_t* tmp_k, uint32_t* tmp_v,
                      uint64_t n, int begin, int end);
void radix_sort_pairs(splatt_ctx* ctx, const uint64_t* src_k, const uint64_t* src_v,
                      uint64_t* out_k, uint64_t* out_v, uint64_t* tmp_k, uint64_t* tmp_v,
                      uint64_t n, int begin, int end);
void radix_sort_pairs(splatt_ctx* ctx, const uint32_t* src_k, const uint32_t* src_v,
                      uint32_t* out_k, uint32_t* out_v, uint32_t* tmp_k, uint32_t* tmp_v,
                      uint64_t n, int begin, int end);

// Ensure the chunk table for `chunk` leaves per work unit exists.
void ensure_chunk_table(splatt_ctx* ctx, DevCsf& c, int chunk);

// Enqueue the validation: *d_bad (device int) becomes nonzero iff some index >= its dim.
void validate_coo_enqueue(splatt_ctx* ctx, const uint32_t* const* d_ind, uint64_t nnz, int N,
                          const uint64_t* dims, int* d_bad);

// Device validation: returns true iff every ind[m][p] < dims[m]  (synchronises).
bool validate_coo_device(splatt_ctx* ctx, const uint32_t* const* d_ind, uint64_t nnz, int N,
                         const uint64_t* dims);

}  // namespace sb

struct splatt_csf {
  int N = 0;
  uint64_t dims[SPLATT_MAX_NMODES] = {0};
  int policy = SPLATT_CSF_ALL;
  int ncsf = 0;
  std::unique_ptr<sb::DevCsf> csf[SPLATT_MAX_NMODES];
  int mode_csf[SPLATT_MAX_NMODES] = {0};    // CSF used for mode n's MTTKRP
  int mode_level[SPLATT_MAX_NMODES] = {0};  // level of mode n in that CSF
  splatt_ctx* ctx = nullptr;
};
