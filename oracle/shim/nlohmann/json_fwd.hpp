// TEST INFRASTRUCTURE ONLY — the reference's tiler.hpp:5 includes
// <nlohmann/json_fwd.hpp>; only the full single-header json.hpp 3.11.3 is on
// disk (cudnn_frontend/thirdparty), which declares everything json_fwd does.
#pragma once
#include <nlohmann/json.hpp>
