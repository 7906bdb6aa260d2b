// npm_net_p16.cu -- instantiation of the decoder kernels for the decoder shape
// n_in=65, width=64, layers=3, 4K=64 (one TU per shape so the heavily
// unrolled kernels compile in parallel).
#include "npm_tc_kernels.cuh"

namespace npm {
using NetT = detail::Net<65, 64, 3, 64>;
int net_smem_p16() { return NetT::SMEM_FLOATS * (int)sizeof(float); }
int net_query_tc_p16(const QueryArgs& a, int sms, cudaStream_t st) { return tck::TcLaunch<NetT>::query(a, sms, st); }
int net_train_tc_p16(const TrainArgs& a, int sms, cudaStream_t st) { return tck::TcLaunch<NetT>::train(a, sms, st); }
}  // namespace npm
