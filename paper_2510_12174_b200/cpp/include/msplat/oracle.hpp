// msplat C++ drop-in -- verification helpers used by the reference tests
// (subset of proj/core/include/msplat/oracle.hpp): the untiled brute-force
// renderer and central finite differences, host double precision.
#pragma once

#include "msplat/rasterizer.hpp"

#include <functional>

namespace msplat {

MultimodalFrame brute_force_render(const Scene& scene, const CameraView& view, const RenderConfig& cfg);

VecX finite_diff(const std::function<Scalar(const VecX&)>& f, const VecX& theta, Scalar eps);

}  // namespace msplat
