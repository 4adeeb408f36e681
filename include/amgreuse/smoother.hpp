// compatibility path of the reference header proj/include/amgreuse/smoother.hpp
#pragma once
#include "../amgreuse_gpu.hpp"
