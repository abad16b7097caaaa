// gsa/gsa.hpp — umbrella header of the B200 GSA operator API (the drop-in for
// the reference's proj/include/gsa/*.hpp). Link with -lgsa_sm100 -lcudart.
#pragma once

#include "gsa/compression.hpp"
#include "gsa/device.hpp"
#include "gsa/errors.hpp"
#include "gsa/gradients.hpp"
#include "gsa/layer.hpp"
#include "gsa/layout.hpp"
#include "gsa/selection.hpp"
#include "gsa/tensor.hpp"
#include "gsa/types.hpp"
#include "gsa/workload.hpp"
