// compatibility path of the reference header proj/include/amgreuse/dense_lu.hpp
#pragma once
#include "../amgreuse_gpu.hpp"
