// SPDX-License-Identifier: Apache-2.0
//
// chunktrain/config.hpp — ModelConfig / AttentionMode (config.hpp:19-49, validate config.cpp:30-51)
// from the facade. Source-compatibility header: see chunktrain/common.hpp.
#pragma once

#include "chunktrain/common.hpp"

namespace chunktrain {
using oomb::AttentionMode;
using oomb::ModelConfig;
}  // namespace chunktrain
