// shard.cuh — clusters of a stage sharded over GPUs,
// each rank holding only the columns it owns.
//
// One process per GPU.  Rank r's matrix is a slab: a full-width Csc whose
// entries are the columns r owns (all rows); nothing is replicated but the
// O(n) metadata (stage numbering, active set, RNG stream).  Per stage:
//   * Clustering: norms of a column by its owner; the m anchor columns are
//     gathered to every rank (gather_columns); each rank scores the pool
//     columns it owns on its slab plus the anchors with the one-GPU kernels,
//     and the assignment (and the repair's score table) meet by an
//     allreduce(max).  The device control path (round-robin, repair, cluster
//     lists) then runs on every rank on identical data.
//   * Reblock: every rank relabels its own slab (ids of the new partition,
//     retired ids dropped); the new clusters are split into W contiguous
//     ranges of about equal cost (shard_ranges, cost c_u^2 + 64 nnz_u with
//     nnz summed over ranks), and redistribute() moves each column to the
//     owner of its new cluster: an all-to-all of column lengths and entries
//     (ncclSend/ncclRecv), ~12 B x nnz/W per rank and stage.
//   * Gram tiles and the pivot search of a cluster read only its columns:
//     each rank searches its clusters.  Exchange 1: the rotation slots and
//     per-cluster counts, each rank's contiguous segment broadcast in place.
//   * Column pass: a rotation mixes columns of its own cluster, so rank r
//     rotates its owned columns with its own rotations.  The transpose of
//     that slab has rows = owned ids and all N columns; the row pass (all
//     rotations, now known to every rank) rotates those partial columns, and
//     row g of it is column g of A'' for the owned retired ids g — the
//     residual masses of rank r's eliminations are complete locally.  The
//     second transpose gives the owned columns of A'': the next stage's slab.
//     The owned eliminations' masses / diagonals are broadcast (small).
// Every value is computed by exactly the kernels of the one-GPU path on the
// same entries in the same order, so the result is bit-identical for any W.
//
// Comm::virt runs W ranks one after another inside one process on one GPU
// (the exchanges become buffer moves): the parity tests use it to prove the
// decomposition bit-exact on a single device.
#pragma once

#include <utility>
#include <vector>

#include "engine.cuh"

struct ncclComm;

namespace pmmf_b200 {

struct Comm {
  int rank = 0;        // this process's rank
  int size = 1;        // ranks in the job (W)
  bool virt = false;   // W virtual ranks in this process, no NCCL
  ncclComm* nccl = nullptr;
  int device = 0;
  int world() const { return size; }
  // NCCL collectives run (also for a one-rank NCCL communicator, which
  // exercises the exchange code on a single GPU)
  bool multi_process() const { return nccl != nullptr; }
  // ranks whose work runs in this process
  std::vector<int> local_ranks() const {
    std::vector<int> r;
    if (virt) {
      for (int i = 0; i < size; ++i) r.push_back(i);
    } else {
      r.push_back(rank);
    }
    return r;
  }
};

// Contiguous split of clusters [0, nclu) into W ranges of about equal cost:
// returns lo[0..W] (lo[0] = 0, lo[W] = nclu).  cost_u = c_u^2 (Gram tile +
// search) + kApplyWeight * nnz_u (rotation passes).  Pure host code.
std::vector<i64> shard_ranges(const std::vector<i64>& cluster_size, const std::vector<i64>& cluster_nnz, int W);

// nnz of every cluster's columns: A.ptr sampled at the cluster offsets.
std::vector<i64> cluster_ptr(const Csc& a, const std::vector<i64>& off, cudaStream_t s);

// In-place broadcast of rank r's segment [seg[r], seg[r+1]) of a device
// array of elements of `elem` bytes, for every r (NCCL, grouped).  No-op
// for one process.
void bcast_segments(void* dev, size_t elem, const std::vector<i64>& seg, const Comm& c, cudaStream_t s);
// max over ranks of one device int32 (no-op for one process).
void allreduce_max_i32(int32_t* dev, const Comm& c, cudaStream_t s);
void allreduce_max_i32(int32_t* dev, i64 n, const Comm& c, cudaStream_t s);

// ---- owned-column slabs -------------------------------
// A slab is a full-width Csc (N columns, rows over all N ids) whose entries
// lie in the column range its rank owns; the other columns are empty.

// sum / max over ranks of device arrays (no-op for one process; virtual
// ranks write disjoint parts of one buffer instead).
void allreduce_sum_i64(int64_t* dev, i64 n, const Comm& c, cudaStream_t s);
void allreduce_sum_f64(double* dev, i64 n, const Comm& c, cudaStream_t s);
void allreduce_max_f64(double* dev, i64 n, const Comm& c, cudaStream_t s);

// out = the columns [c0, c1) of a (full width).
void slab_of(Csc& out, const Csc& a, i64 c0, i64 c1, cudaStream_t s);

// Columns cols[0..m) (stage ids, device) gathered from their owners into
// every rank: a full-width Csc holding exactly those columns.  slabs[i] is
// local rank i's slab, owning [own[i], own[i+1]) ... given as pairs.
void gather_columns(Csc& out, const std::vector<const Csc*>& slabs,
                    const std::vector<std::pair<i64, i64>>& own, const int32_t* cols, int m, i64 N,
                    const Comm& c, cudaStream_t s);

// out = a with b's columns added where a's are empty (full width).
void merge_columns(Csc& out, const Csc& a, const Csc& b, cudaStream_t s);

// The all-to-all reblock exchange: slabs[i] (local rank i, any columns) are
// replaced by the slabs of the new ownership, rank r holding exactly the
// columns [dest[r], dest[r+1]) gathered from every rank (ncclSend/ncclRecv
// across processes; buffer moves between virtual ranks).  Every column
// comes from exactly one source, entries are copied unchanged.
void redistribute(std::vector<Csc>& slabs, const std::vector<i64>& dest, i64 N, const Comm& c, cudaStream_t s);

}  // namespace pmmf_b200
