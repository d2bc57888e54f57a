// Forwarding header: the reference test suites include "servesim/workload.h";
// the B200 drop-in declares the whole API in one header.
#pragma once
#include "nx_servesim.hpp"
