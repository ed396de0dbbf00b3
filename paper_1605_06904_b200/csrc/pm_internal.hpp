// pm_internal.hpp — declarations shared by the host logic, the kernels and the C-ABI layer.
#pragma once
#include <cstdint>
#include <string>

#include "../../include/pm_b200.h"

namespace pm {

// Thread-local status message behind pm_last_error().
int set_error(int code, const std::string& msg);
void clear_error();

// ProjectionPlan validation (projection.hpp:36-52).
int validate_plan(int l, const int32_t* kept, int k);

// 4^k saturating at UINT64_MAX for k >= 32 (detail::pow_sigma, kmer.hpp:33-39).
uint64_t pow4(int k);

// pm_trial_plan for n consecutive trials (kept: n x k), four PRNG seed chains advanced at a time: the chain is a
// dependent multiply-xor recurrence, so interleaving independent trials is what makes it fast on the host.
int trial_plans(int l, int k, uint64_t master, int64_t first_trial, int n, int32_t* kept);

}  // namespace pm
