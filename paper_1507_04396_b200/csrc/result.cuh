// result.cuh — host materialisation of MmfFactorization
// (factorizer.hpp:56-118) and FactorizeStats (:86-109).
#pragma once

#include <array>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace pmmf_b200 {

struct Result {
  struct Stage {
    std::vector<i64> off, members, bypassed;  // partition (bypass cluster last), bypassed ids
    std::vector<i64> rot_idx;                 // R x k global ids, cluster-major
    std::vector<double> rot_q;                // R x k x k row-major
    std::vector<i64> elim_idx;                // stage elimination order
    std::vector<double> elim_diag, elim_mass;
  };
  i64 n = 0;
  int k = 2;
  double residual_sq = 0.0;
  bool trivial = false;
  std::vector<i64> hist;
  std::vector<Stage> stages;
  std::vector<i64> core_idx;
  std::vector<double> core;  // g x g row-major
  std::vector<std::pair<i64, double>> diag;
  double phases[6] = {0, 0, 0, 0, 0, 0};
  pmmf_b200_params params{};  // MmfFactorization::params (factorizer.hpp:117)
  std::vector<std::array<i64, 7>> info;
};

// container.cpp: save_factorization / load_factorization (serialize.hpp)
std::string factorization_to_json(const Result& r);
std::unique_ptr<Result> factorization_from_json(const char* text, size_t len);
void save_factorization(const Result& r, const std::string& path);
std::unique_ptr<Result> load_factorization(const std::string& path);
// Range checks on a result built outside factorize (PMMF_DATA on failure).
void validate_result(const Result& r);

struct Comm;
// comm == nullptr: one GPU (shard.cuh for the sharded decomposition).
std::unique_ptr<Result> factorize_device(const pmmf_b200_coo* in, const pmmf_b200_params& p,
                                         const Comm* comm = nullptr);

}  // namespace pmmf_b200
