// compatibility path of the reference header proj/include/amgreuse/bicgstab.hpp
#pragma once
#include "../amgreuse_gpu.hpp"
