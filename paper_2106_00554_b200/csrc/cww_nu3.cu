#define CWW_NU 3
#include "cww_nu_impl.cuh"
