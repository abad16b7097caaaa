// gsa/workload.hpp — the part of the reference's proj/include/gsa/workload.hpp on
// the hot path's reporting side: selection_sparsity (declared at workload.hpp:112
// but never defined in the reference; semantics from SPEC.md:469-477). The
// workload generator and config parser of that header are test fixtures here
// (oracle/, tests/golden/), not part of the drop-in.
#pragma once

#include "gsa/device.hpp"
#include "gsa/layout.hpp"
#include "gsa/types.hpp"

namespace gsa {

// 1 - (fine keys attended per image query) / image_tokens, attended =
// (|forced windows| + min(k, selectable windows)) * s^2: on a uniform-score
// instance the dynamic picks are the lowest-index non-forced windows, so the
// forced and dynamic sets never overlap (the plan's own dedup is a no-op).
inline double selection_sparsity(const TokenLayout& layout, const GsaParams& params) {
    const gsa_layout lc = device::c_layout(layout);
    const gsa_params pc = device::c_params(params);
    double s = 0.0;
    device::check(gsa_selection_sparsity(&lc, &pc, &s));
    return s;
}

}  // namespace gsa
