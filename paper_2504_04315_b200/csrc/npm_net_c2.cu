// npm_net_c2.cu -- instantiation of the decoder kernels for the decoder shape
// n_in=32, width=64, layers=3, 4K=32 (one TU per shape so the heavily
// unrolled kernels compile in parallel).
#include "npm_tc_kernels.cuh"

namespace npm {
using NetT = detail::Net<32, 64, 3, 32>;
int net_smem_c2() { return NetT::SMEM_FLOATS * (int)sizeof(float); }
int net_query_tc_c2(const QueryArgs& a, int sms, cudaStream_t st) { return tck::TcLaunch<NetT>::query(a, sms, st); }
int net_train_tc_c2(const TrainArgs& a, int sms, cudaStream_t st) { return tck::TcLaunch<NetT>::train(a, sms, st); }
}  // namespace npm
