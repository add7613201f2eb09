#define CWW_NU 2
#include "cww_nu_impl.cuh"
