// compatibility path of the reference header proj/include/amgreuse/hierarchy.hpp
#pragma once
#include "../amgreuse_gpu.hpp"
