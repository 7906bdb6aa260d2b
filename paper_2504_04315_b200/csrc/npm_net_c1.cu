// npm_net_c1.cu -- instantiation of the decoder kernels for the decoder shape
// n_in=16, width=32, layers=2, 4K=32 (one TU per shape so the heavily
// unrolled kernels compile in parallel).
#include "npm_tc_kernels.cuh"

namespace npm {
using NetT = detail::Net<16, 32, 2, 32>;
int net_smem_c1() { return NetT::SMEM_FLOATS * (int)sizeof(float); }
int net_query_tc_c1(const QueryArgs& a, int sms, cudaStream_t st) { return tck::TcLaunch<NetT>::query(a, sms, st); }
int net_train_tc_c1(const TrainArgs& a, int sms, cudaStream_t st) { return tck::TcLaunch<NetT>::train(a, sms, st); }
}  // namespace npm
