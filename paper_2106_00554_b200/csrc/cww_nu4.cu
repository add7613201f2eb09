#define CWW_NU 4
#include "cww_nu_impl.cuh"
