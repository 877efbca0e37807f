// Explicit instantiation of the operator launchers for one degree (SEM_N).
#include "sem1d_launch.cuh"

#ifndef SEM_N
#error "compile with -DSEM_N=<degree>"
#endif

namespace sem1d {
template cudaError_t launch_apply<SEM_N>(const PlanView&, int, const Args&, cudaStream_t);
template cudaError_t launch_ens_forward<SEM_N>(const PlanView&, const EnsArgs&, cudaStream_t);
template cudaError_t launch_ens_adjoint<SEM_N>(const PlanView&, const EnsAdjArgs&, cudaStream_t);
template cudaError_t launch_tile_step<SEM_N>(const PlanView&, int, TileStepArgs, cudaStream_t);
}
