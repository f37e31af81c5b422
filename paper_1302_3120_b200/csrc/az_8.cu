#include "az.cuh"
namespace cssar {
template cudaError_t az_dispatch_mode<8>(int, int, const AzArgs&, cudaStream_t);
}  // namespace cssar
