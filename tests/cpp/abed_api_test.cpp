// Drop-in API tests: the assertions of the reference's own suites
// (/root/reference/proj/tests/{tensor,convolution,checksum,faults,abft_gemm}_test.cpp),
// restated against include/abed/*.hpp, whose compute runs on the B200.
// "Host*" suites touch no device (run on CPU); the rest need a GPU.
#include <abed/abed.hpp>

#include "mini_gtest.hpp"

using namespace abed;

namespace {
Tensor4D random_i8(Dims4 d, SplitMix64& rng) {
  Tensor4D t(d, ElemKind::I8);
  fill_random_i8(t, rng);
  return t;
}
Tensor4D ones_twos_filters() {
  Tensor4D f = Tensor4D::filled({2, 1, 3, 3}, ElemKind::I8, 1);
  for (std::int64_t i = 9; i < 18; ++i) f.view<std::int8_t>()[static_cast<std::size_t>(i)] = 2;
  return f;
}
// straightforward triple loop (test-local, independent of the library)
Tensor4D naive_conv(const Tensor4D& x, const Tensor4D& f, const LayerShape& ls) {
  Tensor4D out(ls.output_dims(), ElemKind::I32);
  for (std::int64_t n = 0; n < ls.n; ++n)
    for (std::int64_t k = 0; k < ls.k; ++k)
      for (std::int64_t p = 0; p < ls.p; ++p)
        for (std::int64_t q = 0; q < ls.q; ++q) {
          std::int32_t acc = 0;
          std::int64_t i = 0;
          for_each_patch_element(x, ls, n, p, q, [&](std::int64_t, std::int64_t, std::int64_t, std::int8_t v) {
            acc += v * f.view<const std::int8_t>()[static_cast<std::size_t>(k * ls.crs() + i++)];
          });
          out.at<std::int32_t>(n, k, p, q) = acc;
        }
  return out;
}
}  // namespace

// ------------------------------------------------------------------ host-only (tensor_test.cpp)
TEST(HostTensor, FilledConstantAndRange) {
  const Tensor4D t = Tensor4D::filled({1, 1, 3, 3}, ElemKind::I8, 1);
  ASSERT_EQ(t.count(), 9);
  for (auto v : t.view<const std::int8_t>()) EXPECT_EQ(v, 1);
  EXPECT_THROW(Tensor4D::filled({1, 1, 1, 1}, ElemKind::I8, 200), std::invalid_argument);
  EXPECT_THROW(Tensor4D::filled({1, 1, 1, 1}, ElemKind::I8, 1.5), std::invalid_argument);
  EXPECT_THROW(Tensor4D({0, 1, 1, 1}, ElemKind::I8), std::invalid_argument);
  Tensor4D u({1, 1, 2, 2}, ElemKind::I32);
  EXPECT_THROW(u.view<std::int8_t>(), std::invalid_argument);
  EXPECT_THROW(u.flat_index(1, 0, 0, 0), std::out_of_range);
  EXPECT_EQ(u.flat_index(0, 0, 1, 1), 3);
}

TEST(HostLayerShape, DerivedExtentsAndGuards) {
  const LayerShape ls = LayerShape::make(1, 3, 8, 8, 4, 3, 3, 2, 2, 1, 1);
  EXPECT_EQ(ls.p, 4);
  EXPECT_EQ(ls.q, 4);
  EXPECT_EQ(ls.crs(), 27);
  EXPECT_THROW(LayerShape::make(1, 1, 3, 3, 1, 5, 3), std::invalid_argument);
  EXPECT_THROW(LayerShape::make(1, 1, 3, 3, 1, 3, 3, 0, 1), std::invalid_argument);
  EXPECT_EQ(capped_spatial(LayerShape::make(1, 8, 1080, 1920, 8, 3, 3, 1, 1, 1, 1), 64).p, 64);
}

TEST(HostPatch, PaddingHalo) {
  const LayerShape ls = LayerShape::make(1, 1, 3, 3, 1, 3, 3, 1, 1, 1, 1);
  const Tensor4D x = Tensor4D::filled(ls.input_dims(), ElemKind::I8, 1);
  const auto e = patch_accumulate_view(x, ls, 0, 0, 0);
  ASSERT_EQ(e.size(), std::size_t{9});
  for (const auto& p : e) EXPECT_EQ(p.value, (p.r == 0 || p.s == 0) ? 0 : 1);
}

TEST(HostSerialize, RoundTripAndMalformed) {
  SplitMix64 rng(5);
  Tensor4D t({2, 3, 4, 5}, ElemKind::I8);
  fill_random_i8(t, rng);
  EXPECT_TRUE(deserialize(serialize(t)) == t);
  auto bytes = serialize(t);
  EXPECT_EQ(bytes.size(), std::size_t{21 + 120});
  bytes[0] = 'X';
  EXPECT_THROW(deserialize(bytes), std::runtime_error);
}

TEST(HostRng, SplitMixAndDeriveSeed) {
  SplitMix64 a(123);
  std::int8_t first[5];
  for (auto& v : first) v = a.next_i8();
  EXPECT_EQ(first[0], 43);  // matches oracle/_ref (tests/test_oracle_golden.py)
  EXPECT_EQ(first[1], 124);
  EXPECT_EQ(derive_seed(7, 1), 7759908279056471943ULL);
}

TEST(HostFlipBit, SingleBitTwosComplementAndBounds) {
  Tensor4D t = Tensor4D::filled({1, 1, 1, 2}, ElemKind::I8, 0);
  EXPECT_EQ(flip_bit(t, 0, 0).view<const std::int8_t>()[0], 1);
  EXPECT_EQ(flip_bit(Tensor4D::filled({1, 1, 1, 1}, ElemKind::I8, -1), 0, 7).view<const std::int8_t>()[0], 127);
  Tensor4D w({1, 1, 2, 2}, ElemKind::I32);
  EXPECT_THROW(flip_bit(w, 4, 0), std::out_of_range);
  EXPECT_THROW(flip_bit(w, 0, 32), std::out_of_range);
}

TEST(HostDecompose, KnownPatternRoundTrip) {
  const auto d = decompose_value(0x12345678);
  EXPECT_EQ(static_cast<std::uint8_t>(d[0]), 0x78);
  EXPECT_EQ(static_cast<std::uint8_t>(d[3]), 0x12);
  for (std::int64_t v : {0LL, -2147483648LL, 2147483647LL, -1LL, 255LL, 256LL})
    EXPECT_EQ(recombine_value(decompose_value(static_cast<std::int32_t>(v))), v);
}

// ------------------------------------------------------------------ device (convolution_test.cpp)
TEST(ConvDirect, OnesWindowCountAndScaling) {
  const LayerShape ls = LayerShape::make(1, 1, 3, 3, 2, 3, 3);
  const Tensor4D out = conv_direct(Tensor4D::filled(ls.input_dims(), ElemKind::I8, 1), ones_twos_filters(), ls);
  EXPECT_EQ(out.view<const std::int32_t>()[0], 9);
  EXPECT_EQ(out.view<const std::int32_t>()[1], 18);
}

TEST(ConvDirect, MatchesBruteForceAndGuards) {
  SplitMix64 rng(21);
  const LayerShape ls = LayerShape::make(2, 4, 8, 8, 3, 3, 3, 2, 2, 1, 1);
  const Tensor4D x = random_i8(ls.input_dims(), rng), f = random_i8(ls.filter_dims(), rng);
  EXPECT_TRUE(conv_direct(x, f, ls) == naive_conv(x, f, ls));
  const LayerShape wide = LayerShape::make(1, 131072, 1, 1, 1, 1, 1);
  EXPECT_THROW(conv_direct(Tensor4D(wide.input_dims(), ElemKind::I8), Tensor4D(wide.filter_dims(), ElemKind::I8), wide),
               std::invalid_argument);
  EXPECT_THROW(conv_direct(Tensor4D::filled({1, 1, 4, 4}, ElemKind::I8, 1), Tensor4D({1, 1, 3, 3}, ElemKind::I8),
                           LayerShape::make(1, 1, 3, 3, 1, 3, 3)),
               std::invalid_argument);
}

TEST(ConvFastPath, EquivalentToBruteForceOnRandomShapes) {
  SplitMix64 rng(43);
  for (int it = 0; it < 12; ++it) {
    const LayerShape ls = LayerShape::make(1 + static_cast<std::int64_t>(rng.below(2)), 1 + static_cast<std::int64_t>(rng.below(5)),
                                           3 + static_cast<std::int64_t>(rng.below(8)), 3 + static_cast<std::int64_t>(rng.below(8)),
                                           1 + static_cast<std::int64_t>(rng.below(5)), 3, 3,
                                           1 + static_cast<std::int64_t>(rng.below(2)), 1 + static_cast<std::int64_t>(rng.below(2)),
                                           static_cast<std::int64_t>(rng.below(2)), static_cast<std::int64_t>(rng.below(2)));
    const Tensor4D x = random_i8(ls.input_dims(), rng), f = random_i8(ls.filter_dims(), rng);
    EXPECT_TRUE(detail::conv_fast_i8(x, f, ls) == naive_conv(x, f, ls));
    EXPECT_TRUE(conv_via_gemm(x, f, ls) == conv_direct(x, f, ls));
  }
}

TEST(Epilog, KnownAnswersAndGuards) {
  EpilogParams relu{1.0f, {0.0f}, Activation::ReLU, ElemKind::I8};
  EXPECT_EQ(epilog(Tensor4D::filled({1, 1, 1, 1}, ElemKind::I32, 9), relu).view<const std::int8_t>()[0], 9);
  EXPECT_EQ(epilog(Tensor4D::filled({1, 1, 1, 1}, ElemKind::I32, -5), relu).view<const std::int8_t>()[0], 0);
  EpilogParams sat{1.0f, {0.5f}, Activation::ReLU, ElemKind::I8};
  EXPECT_EQ(epilog(Tensor4D::filled({1, 1, 1, 1}, ElemKind::I32, 300), sat).view<const std::int8_t>()[0], 127);
  EpilogParams ident{0.5f, {0.0f}, Activation::Identity, ElemKind::I8};
  EXPECT_EQ(epilog(Tensor4D::filled({1, 1, 1, 1}, ElemKind::I32, -5), ident).view<const std::int8_t>()[0], -2);
  EpilogParams f32{0.25f, {0.5f, -100.0f}, Activation::Identity, ElemKind::F32};
  const Tensor4D o = epilog(Tensor4D::filled({1, 2, 1, 1}, ElemKind::I32, 10), f32);
  EXPECT_FLOAT_EQ(o.view<const float>()[0], 3.0f);
  EXPECT_FLOAT_EQ(o.view<const float>()[1], -97.5f);
  EXPECT_THROW(epilog(Tensor4D::filled({1, 2, 1, 1}, ElemKind::I32, 10), relu), std::invalid_argument);
  // FMA probe: the reference's -march=native build yields 35
  EpilogParams probe{0x1.cbe6dap-11f, {0x1.b8ccccp+5f}, Activation::ReLU, ElemKind::I8};
  EXPECT_EQ(epilog(Tensor4D::filled({1, 1, 1, 1}, ElemKind::I32, -21774), probe).view<const std::int8_t>()[0], 35);
}

TEST(FusedConvEpilog, TapsOffIdenticalAndChecksumWorkedExample) {
  SplitMix64 rng(61);
  const LayerShape ls = LayerShape::make(2, 3, 6, 6, 4, 3, 3, 1, 1, 1, 1);
  const Tensor4D x = random_i8(ls.input_dims(), rng), f = random_i8(ls.filter_dims(), rng);
  EpilogParams params{0.05f, {0.1f, -0.2f, 0.3f, 0.0f}, Activation::ReLU, ElemKind::I8};
  const auto fused = fused_conv_epilog(x, f, ls, params);
  EXPECT_TRUE(fused.output == epilog(conv_direct(x, f, ls), params));
  EXPECT_FALSE(fused.output_checksum.has_value());
  const LayerShape l2 = LayerShape::make(1, 1, 3, 3, 2, 3, 3);
  FusedTaps taps;
  taps.output_checksum = true;
  const auto r = fused_conv_epilog(Tensor4D::filled(l2.input_dims(), ElemKind::I8, 1), ones_twos_filters(), l2,
                                   EpilogParams{1.0f, {0.0f, 0.0f}, Activation::ReLU, ElemKind::I8}, taps);
  ASSERT_TRUE(r.output_checksum.has_value());
  EXPECT_EQ(*r.output_checksum, 27);
}

// ------------------------------------------------------------------ device (checksum_test.cpp)
TEST(FilterChecksum, OnesPlusTwosAndPlanes) {
  const FilterChecksum fc = gen_filter_checksum_decomposed(ones_twos_filters());
  for (auto v : fc.sums.view<const std::int32_t>()) EXPECT_EQ(v, 3);
  ASSERT_TRUE(fc.decomposed.has_value());
  EXPECT_EQ((*fc.decomposed)[0].view<const std::int8_t>()[0], 3);
}

TEST(FcVerify, WorkedExampleAndFlip) {
  const LayerShape ls = LayerShape::make(1, 1, 3, 3, 2, 3, 3);
  const Tensor4D x = Tensor4D::filled(ls.input_dims(), ElemKind::I8, 1);
  Tensor4D conv = conv_direct(x, ones_twos_filters(), ls);
  const FilterChecksum fc = gen_filter_checksum_decomposed(ones_twos_filters());
  const Tensor4D extra = recombine_extra_fmaps(conv_checksum_planes(x, ls, *fc.decomposed));
  EXPECT_EQ(extra.view<const std::int64_t>()[0], 27);
  EXPECT_TRUE(fc_verify(conv, extra).pass());
  EXPECT_TRUE(conv_filter_checksum(x, ls, fc) == extra);
  conv.view<std::int32_t>()[0] ^= 1 << 4;
  const VerifyOutcome bad = fc_verify(conv, extra);
  EXPECT_FALSE(bad.pass());
  ASSERT_TRUE(bad.locus.has_value());
  EXPECT_EQ((*bad.locus)[0], 0);
}

TEST(FicVerify, PassFlipAndNegativeControl) {
  SplitMix64 rng(84);
  const LayerShape ls = LayerShape::make(1, 2, 5, 5, 3, 3, 3, 1, 1, 1, 1);
  const Tensor4D x = random_i8(ls.input_dims(), rng), f = random_i8(ls.filter_dims(), rng);
  Tensor4D conv = conv_direct(x, f, ls);
  const std::int64_t expected = fic_dot(gen_filter_checksum(f), gen_input_checksum(x, ls));
  EXPECT_TRUE(fic_verify(conv, expected).pass());
  EXPECT_EQ(fic_verify(conv, expected).lhs, reduce_all_i64(conv));
  conv.view<std::int32_t>()[7] ^= 1 << 12;
  EXPECT_FALSE(fic_verify(conv, expected).pass());
  const LayerShape big = LayerShape::make(1, 64, 16, 16, 64, 3, 3, 1, 1, 1, 1);
  const Tensor4D mx = Tensor4D::filled(big.input_dims(), ElemKind::I8, 127), mf = Tensor4D::filled(big.filter_dims(), ElemKind::I8, 127);
  const Tensor4D mo = detail::conv_fast_i8(mx, mf, big);
  const std::int64_t e = fic_dot(gen_filter_checksum(mf), gen_input_checksum(mx, big));
  EXPECT_EQ(e, 139792236544LL);
  EXPECT_TRUE(fic_verify(mo, e).pass());
  EXPECT_FALSE(fic_verify_forced32(mo, e).pass());
}

TEST(IcVerifyK, ConvOutFlipReportsChannel) {
  SplitMix64 rng(86);
  const LayerShape ls = LayerShape::make(2, 2, 5, 5, 4, 3, 3, 1, 1, 1, 1);
  const Tensor4D x = random_i8(ls.input_dims(), rng), f = random_i8(ls.filter_dims(), rng);
  Tensor4D conv = conv_direct(x, f, ls);
  const InputChecksum ic = gen_input_checksum(x, ls);
  EXPECT_TRUE(ic_verify_k(conv, f, ic).pass());
  conv.view<std::int32_t>()[static_cast<std::size_t>(conv.flat_index(1, 2, 3, 3))] ^= 1 << 9;
  const VerifyOutcome out = ic_verify_k(conv, f, ic);
  EXPECT_FALSE(out.pass());
  ASSERT_TRUE(out.locus.has_value());
  EXPECT_EQ((*out.locus)[0], 2);
}

TEST(IcBatch, DoublingAndOracle) {
  SplitMix64 rng(88);
  const LayerShape ls = LayerShape::make(4, 3, 6, 6, 2, 3, 3, 1, 1, 1, 1);
  const Tensor4D x = random_i8(ls.input_dims(), rng), f = random_i8(ls.filter_dims(), rng);
  const Tensor4D b = ic_batch_checksum(x);
  const Tensor4D conv = conv_direct(x, f, ls);
  EXPECT_TRUE(ic_batch_verify(conv, conv_batch_checksum(b, f, ls)).pass());
  Tensor4D bad = conv;
  bad.view<std::int32_t>()[3] ^= 1 << 2;
  EXPECT_FALSE(ic_batch_verify(bad, conv_batch_checksum(b, f, ls)).pass());
}

TEST(PlanPrecision, TableRows) {
  const PrecisionPlan p = plan_precision(LayerShape::make(1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1), 8);
  EXPECT_EQ(p.bits_output_fmap, 26);
  EXPECT_EQ(p.bits_filter_checksum, 14);
  EXPECT_EQ(p.bits_input_checksum, 20);
  EXPECT_EQ(p.bits_reduced_fic, 43);
  EXPECT_TRUE(p.reduced_fic_kind == ElemKind::I64);
  EXPECT_THROW(plan_precision(LayerShape::make(1, 1, 3, 3, 1, 3, 3), 16), std::invalid_argument);
}

TEST(FloatMode, IntegerValuedDataIsExact) {
  SplitMix64 rng(90);
  const LayerShape ls = LayerShape::make(1, 2, 6, 6, 3, 3, 3, 1, 1, 1, 1);
  Tensor4D x(ls.input_dims(), ElemKind::F32), f(ls.filter_dims(), ElemKind::F32);
  fill_random_f32_integers(x, rng);
  fill_random_f32_integers(f, rng);
  const Tensor4D conv = conv_direct_f32(x, f, ls);
  const double expected = fic_dot_f64(filter_checksum_f64(f), input_checksum_f64(x, ls));
  EXPECT_TRUE(fic_verify_f32(conv, expected, 0.0).pass());
  EXPECT_TRUE(ic_verify_k_f32(conv, f, input_checksum_f64(x, ls), 0.0).pass());
  EXPECT_TRUE(float_verify(1.0, 1.5, 0.5).pass());
  EXPECT_FALSE(float_verify(1.0, 1.5, 0.25).pass());
  EXPECT_THROW(float_verify(0.0, 0.0, -1.0), std::invalid_argument);
}

// ------------------------------------------------------------------ device (faults_test.cpp)
TEST(RunTrial, FcFilterDetectedFcInputNeverDetectedIcFilterEscapes) {
  const LayerShape ls = LayerShape::make(1, 8, 12, 12, 8, 3, 3, 1, 1, 1, 1);
  const Tensor4D x = Tensor4D::filled(ls.input_dims(), ElemKind::I8, 1), f = Tensor4D::filled(ls.filter_dims(), ElemKind::I8, 1);
  EpilogParams p;
  p.scale = 0.05f;
  p.bias.assign(8, 0.0f);
  for (std::uint64_t seed = 1; seed <= 10; ++seed) {
    EXPECT_FALSE(run_trial(ls, x, f, Scheme::FC, InjectionTarget::Filter, p, seed).verify.pass());
    EXPECT_TRUE(run_trial(ls, x, f, Scheme::FC, InjectionTarget::InputFmap, p, seed).verify.pass());
    EXPECT_TRUE(run_trial(ls, x, f, Scheme::IC, InjectionTarget::Filter, p, seed).verify.pass());
    for (auto t : {InjectionTarget::InputFmap, InjectionTarget::Filter, InjectionTarget::ConvOut})
      EXPECT_FALSE(run_trial(ls, x, f, Scheme::FIC, t, p, seed).verify.pass());
  }
  EXPECT_THROW(run_trial(ls, x, f, Scheme::ICBatch, InjectionTarget::Filter, p, 1), std::invalid_argument);
}

TEST(Campaign, AcceptanceCountsAndDeterminism) {
  CampaignConfig c;
  c.shape = LayerShape::make(1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1);
  c.scheme = Scheme::FIC;
  c.target = InjectionTarget::ConvOut;
  c.trials = 1000;
  c.root_seed = 0xC7;
  c.epilog.scale = 0.05f;
  const CampaignReport r = run_campaign(c);
  EXPECT_EQ(r.detected, 928);
  EXPECT_EQ(r.detected_benign, 72);
  EXPECT_EQ(r.sdc, 0);
  EXPECT_EQ(r.detection_rate(), 1.0);
  const CampaignReport a = run_campaign_range(c, 0, 333), b = run_campaign_range(c, 333, 1000);
  EXPECT_EQ(a.detected + b.detected, r.detected);
  c.trials = 0;
  EXPECT_THROW(run_campaign(c), std::invalid_argument);
}

// ------------------------------------------------------------------ abft_gemm_test.cpp
namespace {
Matrix random_matrix(std::int64_t rows, std::int64_t cols, SplitMix64& rng) {
  Matrix m(rows, cols, ElemKind::I8);
  for (auto& v : m.view<std::int8_t>()) v = rng.next_i8();
  return m;
}
}  // namespace

TEST(HostAbftCosts, CostAccounting) {  // abft_gemm_test.cpp:87-98 + the reference's numbers (tests/golden/abft.json)
  const std::int64_t m = 7, n = 5, k = 9;
  const AbftCosts costs = abft_costs(m, n, k);
  EXPECT_EQ(costs.tasks[2].ops, (m + 1) * (n + 1) * k);
  EXPECT_EQ(costs.copy_elements(), m * k + k * n + 2 * m * n);
  EXPECT_EQ(costs.tasks[0].elements_moved, m * k + k * n);
  EXPECT_EQ(costs.tasks[4].elements_moved, 2 * m * n);
  const AbftCosts one_pass = abft_costs(m, n, k, true);
  EXPECT_LT(one_pass.tasks[3].read_bytes, costs.tasks[3].read_bytes);
  EXPECT_EQ(one_pass.tasks[2].ops, costs.tasks[2].ops);
  const std::int64_t want[5][4] = {{0, 108, 432, 108}, {90, 108, 72, 0}, {432, 504, 384, 0}, {82, 768, 8, 0},
                                   {0, 280, 140, 70}};
  for (int t = 0; t < 5; ++t) {
    EXPECT_EQ(costs.tasks[t].ops, want[t][0]);
    EXPECT_EQ(costs.tasks[t].read_bytes, want[t][1]);
    EXPECT_EQ(costs.tasks[t].write_bytes, want[t][2]);
    EXPECT_EQ(costs.tasks[t].elements_moved, want[t][3]);
  }
  EXPECT_EQ(abft_costs(16, 12, 20).copy_elements(), 944);  // cli_test.cpp:143
}

TEST(AbftGemm, IdentityPasses) {
  Matrix eye(2, 2, ElemKind::I8);
  eye.at<std::int8_t>(0, 0) = 1;
  eye.at<std::int8_t>(1, 1) = 1;
  const AbftResult result = abft_gemm(eye, eye);
  EXPECT_TRUE(result.pass());
  EXPECT_EQ(result.c.at<std::int32_t>(0, 0), 1);
  EXPECT_EQ(result.c.at<std::int32_t>(0, 1), 0);
  EXPECT_EQ(result.c.at<std::int32_t>(1, 1), 1);
  EXPECT_EQ(result.c_aug.at<std::int64_t>(2, 2), 2);
}

TEST(AbftGemm, SingleCorruptionFlagsRowAndColumn) {
  SplitMix64 rng(7);
  const Matrix a = random_matrix(6, 5, rng);
  const Matrix b = random_matrix(5, 4, rng);
  AbftResult result = abft_gemm(a, b);
  EXPECT_TRUE(result.pass());
  result.c_aug.at<std::int64_t>(2, 3) ^= std::int64_t{1} << 17;
  const auto [row_check, col_check] = abft_check(result.c_aug);
  EXPECT_FALSE(row_check.pass());
  EXPECT_FALSE(col_check.pass());
  EXPECT_TRUE(row_check.locus.has_value() && (*row_check.locus)[0] == 2);
  EXPECT_TRUE(col_check.locus.has_value() && (*col_check.locus)[0] == 3);
}

TEST(AbftGemm, ChecksumRowMatchesColumnSumOracleAndRandomInstances) {
  SplitMix64 rng(8);
  const Matrix a = random_matrix(8, 8, rng);
  const Matrix b = random_matrix(8, 8, rng);
  const AbftResult result = abft_gemm(a, b);
  EXPECT_TRUE(result.pass());
  for (std::int64_t j = 0; j < 8; ++j) {
    std::int64_t col_sum = 0;
    for (std::int64_t i = 0; i < 8; ++i) {
      std::int64_t c = 0;
      for (std::int64_t t = 0; t < 8; ++t) c += a.at<std::int8_t>(i, t) * b.at<std::int8_t>(t, j);
      EXPECT_EQ(result.c.at<std::int32_t>(i, j), c);
      col_sum += c;
    }
    EXPECT_EQ(result.c_aug.at<std::int64_t>(8, j), col_sum);
  }
  SplitMix64 r9(9);
  for (int iter = 0; iter < 50; ++iter) {
    const std::int64_t m = 1 + static_cast<std::int64_t>(r9.below(16));
    const std::int64_t k = 1 + static_cast<std::int64_t>(r9.below(16));
    const std::int64_t n = 1 + static_cast<std::int64_t>(r9.below(16));
    const Matrix x = random_matrix(m, k, r9), y = random_matrix(k, n, r9);
    EXPECT_TRUE(abft_gemm(x, y).pass());
  }
}

TEST(AbftGemm, Guards) {
  Matrix a(2, 3, ElemKind::I8);
  Matrix b(4, 2, ElemKind::I8);
  EXPECT_THROW(abft_gemm(a, b), std::invalid_argument);
  Matrix a32(2, 2, ElemKind::I32);
  Matrix b32(2, 2, ElemKind::I32);
  EXPECT_THROW(abft_gemm(a32, b32), std::invalid_argument);
}

int main(int argc, char** argv) { return mini_gtest::run_all(argc, argv); }
