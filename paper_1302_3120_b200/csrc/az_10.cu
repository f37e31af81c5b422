#include "az.cuh"
namespace cssar {
template cudaError_t az_dispatch_mode<10>(int, int, const AzArgs&, cudaStream_t);
template size_t az_table_count_t<10>(bool);
template cudaError_t az_table_fill_t<10>(bool, float2*, cudaStream_t);
}  // namespace cssar
