// engine.cuh — device data model of the stage loop and the host entry
// points of each kernel family.
//
// Data layout in HBM:
//   * "stage numbering": id = cluster offset + position in the cluster of
//     the current stage Partition (partition.hpp:19-93).  Row and column ids
//     share it, so block (u,v) of BlockedSparseMatrix (blocked_matrix.hpp:
//     106-118) is the id rectangle [off_u,off_u+1) x [off_v,off_v+1).
//   * Csc: contiguous column-compressed fp64 matrix over stage ids, int32
//     rows sorted ascending inside a column, no stored zeros (value-neutral,
//     SURVEY.md App. A P12).
//   * Paged: the same matrix while rotations rewrite columns: per-column
//     (offset,len) into an append-only arena.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "common.cuh"

namespace pmmf_b200 {

struct Csc {
  i64 N = 0;    // ids
  i64 nnz = 0;
  DBuf<i64> ptr;     // N+1
  DBuf<int32_t> row;
  DBuf<double> val;
};

struct Paged {
  i64 N = 0;
  DBuf<i64> off;      // N
  DBuf<int32_t> len;  // N
  DBuf<int32_t> row;  // arena
  DBuf<double> val;
  i64 cap = 0;
  DBuf<unsigned long long> cursor;  // 1: arena fill
};

// A stage numbering on the device plus its host mirror.
struct Numbering {
  std::vector<i64> s2g, off, g2s;  // host: stage->global, cluster offsets, global->stage (-1)
  DBuf<int32_t> d_blk;             // stage id -> cluster (row block)
  DBuf<int32_t> d_s2g;             // stage id -> global
  DBuf<int32_t> d_g2s;             // global -> stage id (-1 when absent)
  i64 n_global = 0;                // build_device: g2s stays on the device until host_g2s()
  i64 size() const { return static_cast<i64>(s2g.size()); }
  i64 clusters() const { return static_cast<i64>(off.size()) - 1; }
  const std::vector<i64>& host_g2s();  // the host mirror of global -> stage, downloaded on first use
  // from host cluster lists (validated: the input partition)
  void build(const std::vector<std::vector<i64>>& clusters, i64 n, cudaStream_t s);
  // from a device member list (a stage partition built on the device) and
  // the cluster offsets; host mirrors are copied back
  void build_device(DBuf<int32_t>&& members, std::vector<i64> offsets, i64 n, cudaStream_t s);
};

// ---- matrix.cu
// from_triplets (blocked_matrix.hpp:138-156) on the device: validates in
// input order, stable-sorts by (col,row), sums duplicates in input order,
// drops exact zeros unless keep_zeros (the reference stores them; only the
// preconditioners' patterns see the difference).  rows/cols/vals are device
// pointers.
void csc_from_coo(Csc& out, const Numbering& nb, i64 n, i64 nnz, const int64_t* rows, const int64_t* cols,
                  const double* vals, cudaStream_t s, bool keep_zeros = false);
// max_asymmetry (blocked_matrix.hpp:447-463) and frobenius_norm_sq.
void csc_symmetry(const Csc& a, const Numbering& nb, double* max_asym, double* fro_sq, cudaStream_t s);
// Paged view of a contiguous matrix (takes ownership of its arrays).
void paged_from_csc(Paged& p, Csc&& a, i64 extra_capacity, cudaStream_t s);
// Transpose of a paged matrix into a contiguous one (stable row sort).
void transpose_paged(Csc& out, const Paged& p, cudaStream_t s);
// Reblock (blocked_matrix.hpp:318-367): ids of `from` relabelled through
// map[old id] -> new id (-1 = dropped), columns gathered, rows re-sorted.
void reblock(Csc& out, const Csc& a, const DBuf<int32_t>& map, const DBuf<int32_t>& new2old, i64 n_new,
             cudaStream_t s);

// ---- cluster.cu
struct ClusterOut {
  // device: the clusters' members (global ids) in DFS order, each cluster
  // ascending, followed by the bypassed columns; sizes[u] per cluster
  DBuf<int32_t> members;
  std::vector<i64> sizes;
  std::vector<i64> bypassed;  // ascending global ids
  int max_depth = 0;
};
// cluster_columns (clustering.hpp:183-225) over the pre-reblock matrix
// (numbering nb); active ascending global ids.
struct Comm;
// The owned-column slabs of this process's ranks (shard.cuh): slabs[i]
// holds the columns [own[i].first, own[i].second) of the matrix.  With one
// slab owning everything and no communicator the clustering is the one-GPU
// path.  Sharded: the norms and scores of a column are computed by its
// owner (the anchor columns gathered to every rank), combined by max.
struct SlabSet {
  std::vector<const Csc*> slabs;
  std::vector<std::pair<i64, i64>> own;
  const Comm* comm = nullptr;
  bool sharded() const { return comm != nullptr; }
};
ClusterOut cluster_columns_dev(const SlabSet& ss, const Numbering& nb, const std::vector<i64>& active, i64 n,
                               i64 m_target, i64 c_min, i64 c_max, int d_max, bool bypass, uint64_t seed,
                               cudaStream_t s);

// ---- gram.cu
// Dense c_u x c_u column-major tiles of G_u (blocked_matrix.hpp:238-254)
// and D_u (:257-266) for clusters [u0,u1) at tile offsets tile_off[u]-tile_off[u0].
void gram_tiles(const Csc& a, const std::vector<i64>& off, i64 u0, i64 u1, const std::vector<i64>& tile_off,
                double* G, double* D, cudaStream_t s);

// ---- search.cu
struct SearchBatch {
  // per cluster u in [u0,u1):
  DBuf<int64_t> c;         // cluster size
  DBuf<int64_t> tile;      // tile offset (elements) into G/D
  DBuf<int64_t> budget;    // elimination cap (factorizer.hpp:463-479)
  DBuf<uint64_t> seed;     // derive(seed,{0xF0,p,u})
  DBuf<int64_t> out_base;  // first rotation / elimination slot
  DBuf<int32_t> order;     // CTA launch order: batch-relative clusters by decreasing size
  std::vector<int64_t> h_c;  // host copy of c
};
struct SearchOut {
  DBuf<int32_t> nrot, nelim;   // per cluster
  DBuf<int32_t> rot_loc;       // R x k local indices
  DBuf<double> rot_q;          // R x k x k
  DBuf<int32_t> rot_level;     // R: dependency level in the apply, 0 = exact identity
  DBuf<int32_t> elim_loc;      // R local indices, elimination order
  DBuf<int32_t> error;         // 1: non-symmetric sub-Gram (invalid_argument)
};
// Clusters [u0, u0+nclusters): per-cluster arrays of b are batch-relative,
// out.nrot/out.nelim are indexed by absolute cluster u, slots are absolute.
void search_clusters(const SearchBatch& b, i64 u0, i64 nclusters, int k, double eta, double* G, double* D,
                     i64 max_c, SearchOut& out, cudaStream_t s);

// ---- apply.cu
// One rotation stream applied to the columns of a paged matrix
// (factorizer.hpp:362-380, sparse.hpp:123-156): rotation t acts on ids
// col_ids[t*k .. t*k+k) with q = rot_q[t]; rotations are grouped in levels
// of mutually independent rotations (level_start).
struct LevelPlan {
  i64 R = 0;                 // rotation slots
  int k = 2;
  int max_level = 0;
  DBuf<int32_t> ids;         // R x k stage ids
  const double* q = nullptr; // R x k x k (non-owning)
  DBuf<int32_t> order;       // slots sorted by level (level-0 slots first, skipped)
  std::vector<i64> level_start;  // host: [level-1 start] for levels 1..max_level, plus end
  std::vector<int32_t> h_order;  // host copy of order
};

// A compact column range [c0, c1) of a matrix (ptr local, starting at 0).
struct Piece {
  i64 c0 = 0, c1 = 0, nnz = 0;
  DBuf<i64> ptr;
  DBuf<int32_t> row;
  DBuf<double> val;
};

// Residual accounting fused into the row pass (factorizer.hpp:521-547):
// the final columns c of the row pass are the rows of A', so row g of them
// is column g of A'.  For retired g the masses sum v^2 over c in ascending
// order (columns are finalised batch by batch, chunk by chunk, in that
// order; the running sums are carried in `mass`), taking c when it survives
// or retires later than g.
struct MassSpec {
  const int32_t* row_rank = nullptr;  // stage id -> elimination rank, -1 if not retired
  const int32_t* col_key = nullptr;   // stage id -> INT_MAX if surviving, else its rank
  double* mass = nullptr;             // by rank (zero-initialised by the caller)
  double* diag = nullptr;             // by rank
  i64 chunk_nnz = 0;                  // entries sorted at once
  i64 n_retired = 0;                  // ranks of the retired rows present: [rank_base, rank_base + n_retired)
  i64 rank_base = 0;                  // (a sharded slab holds only its own clusters' eliminations)
};

// One pass of a stage's rotations over the columns of `in` (stage
// numbering, cluster offsets `off`, rotation slots of cluster u in
// [slot_base[u], slot_base[u+1])), batch by batch of clusters holding at
// most batch_nnz input entries.  The final columns are returned as pieces;
// when keep_row != nullptr, a column c keeps only rows r with keep_row[r]
// unless keep_all_col[c].
// `growth` is the expected arena/input ratio of a batch (final columns plus
// superseded versions); the arena starts at that size so that compactions
// (copy + re-map) stay rare.  With `ms`, the residual masses are taken from
// the final columns before they are filtered into pieces.  Only clusters
// [u_lo, u_hi) are passed (u_hi < 0: all); pieces then cover their columns.
void rotate_pass(std::vector<Piece>& out, const Csc& in, const std::vector<i64>& off,
                 const std::vector<i64>& slot_base, const LevelPlan& plan, const uint8_t* keep_row,
                 const uint8_t* keep_all_col, i64 batch_nnz, double growth, const MassSpec* ms,
                 cudaStream_t s, i64 u_lo = 0, i64 u_hi = -1);
// Transpose of a matrix given as pieces covering [0, N), keeping only rows
// r with keep_row[r] (all when nullptr); sorted in chunks of <= chunk_nnz
// entries so the sort buffers stay bounded.
void transpose_pieces(Csc& out, const std::vector<Piece>& in, i64 N, const uint8_t* keep_row, i64 chunk_nnz,
                      cudaStream_t s);
// Builds the level plan from a search result: slot = out_base[u] + t for
// t < nrot[u]; stage id = cluster_off[u] + local.
void build_plan(LevelPlan& plan, const SearchOut& so, const DBuf<int64_t>& out_base,
                const DBuf<int64_t>& cluster_off, i64 nclusters, i64 R, int k, cudaStream_t s);

}  // namespace pmmf_b200
