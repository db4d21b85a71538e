// Forwarding header: the B200 drop-in API lives in graphfuse.hpp.
#pragma once
#include "graphfuse/graphfuse.hpp"
