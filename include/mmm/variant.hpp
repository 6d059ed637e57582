// Forwarding header: the drop-in declarations live in mmm_b200.hpp.
#pragma once
#include "../mmm_b200.hpp"
