#define CWW_NU 5
#include "cww_nu_impl.cuh"
