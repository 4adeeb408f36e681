// compatibility path of the reference header proj/include/amgreuse/coarsening.hpp
#pragma once
#include "../amgreuse_gpu.hpp"
