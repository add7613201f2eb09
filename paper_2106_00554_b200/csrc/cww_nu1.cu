#define CWW_NU 1
#include "cww_nu_impl.cuh"
