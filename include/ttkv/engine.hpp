// Drop-in forwarding header: the reference module "ttkv/engine.hpp" is provided
// by the B200 implementation in gpu_dropin.hpp.
#pragma once
#include "ttkv/gpu_dropin.hpp"
