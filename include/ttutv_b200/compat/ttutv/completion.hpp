// Forwarding header: code written against the reference include/ttutv/completion.hpp compiles
// unchanged against the B200 engine with -Iinclude/ttutv_b200/compat -Iinclude.
#pragma once
#include "ttutv_b200/ttutv.hpp"
