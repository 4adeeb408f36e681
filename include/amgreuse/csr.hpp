// compatibility path of the reference header proj/include/amgreuse/csr.hpp
#pragma once
#include "../amgreuse_gpu.hpp"
