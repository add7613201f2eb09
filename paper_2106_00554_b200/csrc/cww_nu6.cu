#define CWW_NU 6
#include "cww_nu_impl.cuh"
