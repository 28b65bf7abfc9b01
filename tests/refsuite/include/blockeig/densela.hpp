// Forwarding header (test infrastructure): the reference suites include "blockeig/densela.hpp";
// this build resolves it to the B200 C++ mirror (include/blockeig_b200.hpp).
#pragma once
#include "blockeig_b200.hpp"
