/*
 * ssa_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU oracle for the StochKit-FF hot path
 * (arxiv/paper_1007_1768): Gillespie direct-method SSA trajectories of a
 * mass-action network, aligned online to a sample grid ("selective memory",
 * PAPER.md:147 §3.2.1) and reduced to per-species mean and variance
 * (PAPER.md:129, :177).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1007_1768_b200/) never includes, links or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 * (x86-64 SSE2 arithmetic, FLT_EVAL_METHOD == 0, round-to-nearest-even;
 * every floating-point operation below is a single IEEE fp64 operation; the
 * only fused operations are the explicit fma() calls of plog, R11).
 *
 * Readings of the paper used here are the ones listed in DESIGN.md §3
 * ("readings"), numbered R1..R30 after SURVEY.md §8(c) Q1..Q30.
 *
 * Parity pins (tests/test_oracle_*.py):
 *   philox  -- equal to curand_Philox4x32_10 (cuRAND header, host-compiled)
 *   u53     -- closed-form endpoints, exactness
 *   plog    -- <= 2 ulp of logl on >= 1e6 inputs; special values
 *   propensity -- SPEC.md:87-88 printed values, C(x,2) closed form
 *   step    -- SPEC.md:174 worked example; frozen-state statistics
 *   aligner -- SPEC.md:250 example restated on a grid (tests/golden)
 *   moments -- SPEC.md:270-272 printed example
 *   trajectory -- closed forms (immigration-death Poisson, pure-death
 *                 binomial), CME by matrix exponential, structural
 *                 invariants of the HIV network (U0 == 1, F nondecreasing).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#if defined(__FLT_EVAL_METHOD__) && __FLT_EVAL_METHOD__ != 0
#error "oracle requires FLT_EVAL_METHOD == 0 (SSE2 double arithmetic)"
#endif

/* ------------------------------------------------------------------------ */
/* Status codes (mirror the meaning of ssa_status in include/ssa.h, but are  */
/* defined here independently).                                              */
/* ------------------------------------------------------------------------ */
enum {
    OR_OK = 0,
    OR_ERR_INVALID = 1,
    OR_ERR_NUMERIC = 3,   /* non-finite propensity      */
    OR_ERR_OVERFLOW = 4,  /* a sampled count > INT32_MAX (R20)    */
};

/* ------------------------------------------------------------------------ */
/* Model (parameters, integer state vector, integer            */
/* stoichiometric matrix, propensity vector).                                */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t S;               /* number of species                          */
    int32_t R;               /* number of reactions                        */
    const int64_t *x0;       /* [S] initial counts           */
    const int32_t *n_reac;   /* [R] number of reactant terms (0..3)        */
    const int32_t *reac_sp;  /* [R*3] reactant species                     */
    const int32_t *reac_coef;/* [R*3] reactant coefficient m >= 1          */
    const int64_t *nu;       /* [R*S] net change, products - reactants     */
    const double *rate;      /* [R] rate constant k_j                      */
    const int32_t *mod_sp;   /* [R] modifier species or -1   */
    const double *mod_coef;  /* [R] modifier coefficient d_j               */
    /* gated propensities (NEXT 3; SPEC.md:424 mu*step(V5)*(1-step(V4))):   */
    const int32_t *mass_action; /* [R] 1: h = prod C(x,m); 0: h = 1        */
    const int32_t *n_gates;  /* [R] number of gates (0..4)                 */
    const int32_t *gate_sp;  /* [R*4] gate species                         */
    const int32_t *gate_kind;/* [R*4] 0: [x > 0] (step), 1: [x == 0]       */
} oracle_model;

typedef struct {
    uint64_t events;     /* applied events (t <= s_K)                        */
    uint64_t hash;       /* FNV-1a style hash of the firing sequence         */
    double t_last;       /* time of the last applied event (0 if none)       */
    uint64_t near_ties;  /* grid crossings with an event within 1e-9 rel.    */
    int32_t absorbed;    /* 1 if a0 == 0 was reached before s_K              */
    int32_t status;      /* OR_OK or error                                   */
    int32_t err_reaction;/* reaction index of a non-finite propensity        */
    int32_t pad;
} oracle_summary;

/* ------------------------------------------------------------------------ */
/* a2: Philox4x32-10 (Salmon et al., SC'11), the counter-based RNG that      */
/* replaces StochKit's non-reentrant sprng (PAPER.md:129, :139 fn.2;         */
/* DESIGN.md R8).  Key = (seed lo, seed hi); counter = (e lo, e hi, id lo,   */
/* id hi).                                                                   */
/* ------------------------------------------------------------------------ */
#define PH_M0 0xD2511F53u
#define PH_M1 0xCD9E8D57u
#define PH_W0 0x9E3779B9u
#define PH_W1 0xBB67AE85u

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)PH_M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)PH_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += PH_W0;
        k1 += PH_W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u53 (R9): the top 52 bits of a 64-bit word mapped to the open
 * interval: u = (w >> 12) * 2^-52 + 2^-53, exactly (2m+1) * 2^-53,
 * in [2^-53, 1 - 2^-53]. */
double oracle_u53(uint64_t w)
{
    double m = (double)(w >> 12);           /* exact: < 2^52 */
    return m * 0x1p-52 + 0x1p-53;           /* both operations exact */
}

/* ------------------------------------------------------------------------ */
/* plog (R11): the pinned natural logarithm both sides implement   */
/* bit-for-bit (round 2: table-driven, no division).  u = 2^e * m, m in      */
/* [1, 2) from the bits; i = the top 7 fraction bits of m (bucket            */
/* [1 + i/128, 1 + (i+1)/128)); for i >= 53 (m >= 1.4140625) m is halved and */
/* e incremented, so m lies in [0.707, 1.414).  Per bucket: c_i its centre   */
/* (1 + (2i+1)/256, halved for i >= 53), inv_i = fl(1/c_i) (inv = 1 for the  */
/* buckets i = 0 and i = 127 that hold m near 1, so ln u near 0 is exact in  */
/* relative terms), T_i = -ln(inv_i) split into T_hi = fl(T_i) and T_lo =    */
/* fl(T_i - T_hi).  Then r = fma(m, inv_i, -1) (|r| <= 2^-7),                */
/* ln(1+r) = r + r^2 Q(r), Q = sum_{k=2..7} (-1)^(k+1) r^(k-2) / k (Horner   */
/* with explicit fma), ln u = fma(e, ln2_hi, T_hi) + (fma(e, ln2_lo, T_lo) + */
/* ln(1+r)).  Defined for positive normal u; <= 1.4 ulp of logl (pinned).    */
/* ------------------------------------------------------------------------ */
static double bits_to_double(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t double_to_bits(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }

/* {inv_i, T_hi, T_lo} for i = 0..127 (pinned against exact arithmetic in tests). */
static const double PLOG_TAB[128][3] = {
        {0x1.0000000000000p+0, 0x0.0p+0, 0x0.0p+0},
        {0x1.fa11caa01fa12p-1, 0x1.7dc475f810a69p-7, 0x1.74944bc161072p-61},
        {0x1.f6310aca0dbb5p-1, 0x1.3cea44346a584p-6, -0x1.865ad48159d00p-61},
        {0x1.f25f644230ab5p-1, 0x1.b9fc027af919ap-6, -0x1.90ae69229dc86p-60},
        {0x1.ee9c7f8458e02p-1, 0x1.1b0d98923d97fp-5, -0x1.74d7444dd6241p-59},
        {0x1.eae807aba01ebp-1, 0x1.58a5bafc8e4d3p-5, -0x1.cab8569c56e40p-64},
        {0x1.e741aa59750e4p-1, 0x1.95c830ec8e3f2p-5, 0x1.eb41d00a417e9p-60},
        {0x1.e3a9179dc1a73p-1, 0x1.d276b8adb0b56p-5, 0x1.078f14c95ff53p-59},
        {0x1.e01e01e01e01ep-1, 0x1.075983598e471p-4, 0x1.006d2999e22dcp-58},
        {0x1.dca01dca01dcap-1, 0x1.253f62f0a1417p-4, 0x1.1f6d34e01d981p-61},
        {0x1.d92f2231e7f8ap-1, 0x1.42edcbea646eep-4, -0x1.511583653349bp-58},
        {0x1.d5cac807572b2p-1, 0x1.60658a93750c4p-4, -0x1.f108b1d8436d3p-59},
        {0x1.d272ca3fc5b1ap-1, 0x1.7da766d7b12d0p-4, 0x1.a2240644d7da2p-59},
        {0x1.cf26e5c44bfc6p-1, 0x1.9ab42462033aep-4, -0x1.a099e1c184e8ep-59},
        {0x1.cbe6d9601cbe7p-1, 0x1.b78c82bb0eda0p-4, -0x1.3ef0e61f9b03cp-58},
        {0x1.c8b265afb8a42p-1, 0x1.d4313d66cb35dp-4, 0x1.b90dd951d90fap-58},
        {0x1.c5894d10d4986p-1, 0x1.f0a30c01162a4p-4, 0x1.8be64b8b7759bp-59},
        {0x1.c26b5392ea01cp-1, 0x1.0671512ca596fp-3, -0x1.2f39b81479b67p-58},
        {0x1.bf583ee868d8bp-1, 0x1.14785846742acp-3, 0x1.94409f1d3f83ap-60},
        {0x1.bc4fd65883e7bp-1, 0x1.2266f190a5acdp-3, -0x1.dab840e7f6177p-57},
        {0x1.b951e2b18ff23p-1, 0x1.303d718e47fd5p-3, -0x1.b5ae71f658247p-57},
        {0x1.b65e2e3beee05p-1, 0x1.3dfc2b0ecc62ap-3, 0x1.ba62b8c13f7f4p-57},
        {0x1.b37484ad806cep-1, 0x1.4ba36f39a55e5p-3, -0x1.f767e433c98aap-57},
        {0x1.b094b31d922a4p-1, 0x1.59338d9982085p-3, 0x1.8d16eaaba9419p-57},
        {0x1.adbe87f94905ep-1, 0x1.66acd4272ad51p-3, -0x1.9201c9c3d5165p-59},
        {0x1.aaf1d2f87ebfdp-1, 0x1.740f8f54037a3p-3, 0x1.6d9bf9d57b326p-58},
        {0x1.a82e65130e159p-1, 0x1.815c0a14357e9p-3, 0x1.141b7f8c5fa9ep-58},
        {0x1.a574107688a4ap-1, 0x1.8e928de886d41p-3, 0x1.2589eb96a6240p-59},
        {0x1.a2c2a87c51ca0p-1, 0x1.9bb362e7dfb85p-3, -0x1.51439c1ff83e7p-58},
        {0x1.a01a01a01a01ap-1, 0x1.a8becfc882f19p-3, -0x1.a8c37918c39ebp-58},
        {0x1.9d79f176b682dp-1, 0x1.b5b519e8fb5a6p-3, -0x1.d5d8023e61e5fp-57},
        {0x1.9ae24ea5510dap-1, 0x1.c2968558c18c2p-3, 0x1.6108e3ae024acp-60},
        {0x1.9852f0d8ec0ffp-1, 0x1.cf6354e09c5ddp-3, 0x1.339a07d55b696p-57},
        {0x1.95cbb0be377aep-1, 0x1.dc1bca0abec7bp-3, 0x1.c698a33316dfbp-58},
        {0x1.934c67f9b2ce6p-1, 0x1.e8c0252aa5a60p-3, -0x1.dc074737f9135p-60},
        {0x1.90d4f120190d5p-1, 0x1.f550a564b7b37p-3, -0x1.13a09202fe73dp-57},
        {0x1.8e6527af1373fp-1, 0x1.00e6c45ad501dp-2, -0x1.3b9568ff6feadp-57},
        {0x1.8bfce8062ff3ap-1, 0x1.071b85fcd590dp-2, 0x1.08b83fcbdef40p-57},
        {0x1.899c0f601899cp-1, 0x1.0d46b579ab74bp-2, 0x1.21f640e1e5ec9p-56},
        {0x1.87427bcc092b9p-1, 0x1.136870293a8b0p-2, 0x1.86cc531dba494p-57},
        {0x1.84f00c2780614p-1, 0x1.1980d2dd4236fp-2, -0x1.02c2e4f1b2eb9p-56},
        {0x1.82a4a0182a4a0p-1, 0x1.1f8ff9e48a2f3p-2, -0x1.93fbf3418960dp-57},
        {0x1.8060180601806p-1, 0x1.2596010df763ap-2, -0x1.9eed8ae0ebd3cp-59},
        {0x1.7e225515a4f1dp-1, 0x1.2b9303ab89d25p-2, -0x1.85ad7f614ab51p-58},
        {0x1.7beb3922e017cp-1, 0x1.31871c9544185p-2, -0x1.ea3598981366fp-57},
        {0x1.79baa6bb6398bp-1, 0x1.3772662bfd85cp-2, 0x1.02a7589fba088p-57},
        {0x1.77908119ac60dp-1, 0x1.3d54fa5c1f710p-2, 0x1.53668e578d9cdp-58},
        {0x1.756cac201756dp-1, 0x1.432ef2a04e813p-2, -0x1.83262e2b59206p-57},
        {0x1.734f0c541fe8dp-1, 0x1.49006804009d0p-2, -0x1.bff0d07c5df6dp-59},
        {0x1.713786d9c7c09p-1, 0x1.4ec9732600269p-2, -0x1.1aa87d977dc5ep-56},
        {0x1.6f26016f26017p-1, 0x1.548a2c3add263p-2, -0x1.58ce7bf1846eep-56},
        {0x1.6d1a62681c861p-1, 0x1.5a42ab0f4cfe2p-2, -0x1.c6bcb7dee9a3dp-56},
        {0x1.6b1490aa31a3dp-1, 0x1.5ff3070a793d4p-2, -0x1.063077d7e37b7p-56},
        {0x1.691473a88d0c0p+0, -0x1.602d08af091ecp-2, -0x1.a45db7cfd9230p-56},
        {0x1.6719f3601671ap+0, -0x1.5a8cadbbedfa1p-2, -0x1.64f5081307f22p-60},
        {0x1.6524f853b4aa3p+0, -0x1.54f431b7be1a8p-2, 0x1.0b3f6ef6ae452p-58},
        {0x1.63356b88ac0dep+0, -0x1.4f637ebba9810p-2, 0x1.68cb3124b9245p-56},
        {0x1.614b36831ae94p+0, -0x1.49da7f3bcc420p-2, 0x1.d964a168ccacbp-57},
        {0x1.5f66434292dfcp+0, -0x1.44591e0539f49p-2, -0x1.a76d6dc2782dap-59},
        {0x1.5d867c3ece2a5p+0, -0x1.3edf463c1683ep-2, 0x1.c852fe587def8p-57},
        {0x1.5babcc647fa91p+0, -0x1.396ce359bbf53p-2, 0x1.5c5663663d163p-59},
        {0x1.59d61f123ccaap+0, -0x1.3401e12aecba0p-2, -0x1.f95523adc5c9fp-57},
        {0x1.5805601580560p+0, -0x1.2e9e2bce12286p-2, 0x1.f3ed72e23e134p-57},
        {0x1.56397ba7c52e2p+0, -0x1.2941afb186b7cp-2, -0x1.6a4678ebaa300p-59},
        {0x1.54725e6bb82fep+0, -0x1.23ec5991eba49p-2, -0x1.76eba35bbf0dfp-61},
        {0x1.52aff56a8054bp+0, -0x1.1e9e1678899f5p-2, -0x1.64b0dd2687939p-58},
        {0x1.50f22e111c4c5p+0, -0x1.1956d3b9bc2f9p-2, -0x1.0e75a3542856fp-58},
        {0x1.4f38f62dd4c9bp+0, -0x1.14167ef367784p-2, -0x1.ef824daaf53e9p-56},
        {0x1.4d843bedc2c4cp+0, -0x1.0edd060b78082p-2, -0x1.2d4b610d7d4f5p-57},
        {0x1.4bd3edda68fe1p+0, -0x1.09aa572e6c6d4p-2, -0x1.f9e17343426a9p-56},
        {0x1.4a27fad76014ap+0, -0x1.047e60cde83b7p-2, -0x1.08869cbf9e344p-56},
        {0x1.4880522014880p+0, -0x1.feb2233ea07cbp-3, -0x1.8de00938b4c30p-61},
        {0x1.46dce34596066p+0, -0x1.f474b134df228p-3, 0x1.9f1df7b5daab7p-60},
        {0x1.453d9e2c776cap+0, -0x1.ea4449f04aaf5p-3, 0x1.f33919ab94074p-57},
        {0x1.43a2730abee4dp+0, -0x1.e020cc6235ab5p-3, 0x1.f0adb91423f18p-57},
        {0x1.420b5265e5951p+0, -0x1.d60a17f903514p-3, 0x1.50df841a71b7ap-57},
        {0x1.40782d10e6566p+0, -0x1.cc000c9db3c52p-3, -0x1.67a2a8500729ep-58},
        {0x1.3ee8f42a5af07p+0, -0x1.c2028ab17f9b5p-3, -0x1.c11aa3853a5f0p-57},
        {0x1.3d5d991aa75c6p+0, -0x1.b811730b823d4p-3, 0x1.d7c46328983c6p-58},
        {0x1.3bd60d9232955p+0, -0x1.ae2ca6f672bd8p-3, 0x1.a4a356155f779p-57},
        {0x1.3a524387ac822p+0, -0x1.a454082e6ab03p-3, 0x1.e0df823a3cb3dp-58},
        {0x1.38d22d366088ep+0, -0x1.9a8778debaa3ap-3, -0x1.28fbfb0e3f0fcp-58},
        {0x1.3755bd1c945eep+0, -0x1.90c6db9fcbcdbp-3, 0x1.357718d7ca4cfp-58},
        {0x1.35dce5f9f2af8p+0, -0x1.871213750e994p-3, 0x1.a97a0ca115d60p-57},
        {0x1.34679ace01346p+0, -0x1.7d6903caf5acdp-3, 0x1.0b17c301d6e14p-57},
        {0x1.32f5ced6a1dfap+0, -0x1.73cb9074fd14dp-3, 0x1.721a000b4cf01p-57},
        {0x1.3187758e9ebb6p+0, -0x1.6a399dabbd383p-3, -0x1.76332bd4b341fp-57},
        {0x1.301c82ac40260p+0, -0x1.60b3100b09474p-3, -0x1.526cee0fd7f4ap-57},
        {0x1.2eb4ea1fed14bp+0, -0x1.5737cc9018cddp-3, 0x1.00b28ef013c72p-57},
        {0x1.2d50a012d50a0p+0, -0x1.4dc7b897bc1c7p-3, -0x1.b60ae1ff0e82ep-59},
        {0x1.2bef98e5a3711p+0, -0x1.4462b9dc9b3dcp-3, 0x1.85388d830c709p-59},
        {0x1.2a91c92f3c105p+0, -0x1.3b08b6757f2a7p-3, -0x1.5e1ad9be0a4cdp-57},
        {0x1.293725bb804a5p+0, -0x1.31b994d3a4f86p-3, 0x1.1238b5efe0665p-57},
        {0x1.27dfa38a1ce4dp+0, -0x1.28753bc11aba2p-3, 0x1.7394d9fa33313p-57},
        {0x1.268b37cd60127p+0, -0x1.1f3b925f25d44p-3, -0x1.08b27be4e6b15p-57},
        {0x1.2539d7e9177b2p+0, -0x1.160c8024b27b0p-3, 0x1.355bfd870afebp-59},
        {0x1.23eb79717605bp+0, -0x1.0ce7ecdccc28bp-3, -0x1.1b57fea88da98p-59},
        {0x1.22a0122a0122ap+0, -0x1.03cdc0a51ec0dp-3, -0x1.19e2d3f8b7d10p-57},
        {0x1.21579804855e6p+0, -0x1.f57bc7d9005dbp-4, 0x1.d361574fb24e2p-58},
        {0x1.2012012012012p+0, -0x1.e3707ee30487bp-4, -0x1.9399d9aaf3b33p-59},
        {0x1.1ecf43c7fb84cp+0, -0x1.d179788219362p-4, 0x1.b12841044a96cp-58},
        {0x1.1d8f5672e4abdp+0, -0x1.bf968769fca18p-4, 0x1.06e4fb7af9c69p-58},
        {0x1.1c522fc1ce059p+0, -0x1.adc77ee5aea8ep-4, -0x1.d7d8f39bee658p-58},
        {0x1.1b17c67f2bae3p+0, -0x1.9c0c32d4d254dp-4, 0x1.627a0e199f569p-58},
        {0x1.19e0119e0119ep+0, -0x1.8a6477a91dc29p-4, 0x1.3d4190a482421p-58},
        {0x1.18ab083902bdbp+0, -0x1.78d02263d82d7p-4, -0x1.cbca5b4fdb87ep-58},
        {0x1.1778a191bd684p+0, -0x1.674f089365a78p-4, -0x1.ca64e9980e048p-59},
        {0x1.1648d50fc3201p+0, -0x1.55e10050e0382p-4, -0x1.9a0629e3973e4p-58},
        {0x1.151b9a3fdd5c9p+0, -0x1.4485e03dbdfb0p-4, -0x1.3ba349aadbc6dp-58},
        {0x1.13f0e8d344724p+0, -0x1.333d7f8183f4ap-4, 0x1.adaa06e211e9ep-59},
        {0x1.12c8b89edc0acp+0, -0x1.2207b5c7854a1p-4, -0x1.b3f0431efb154p-58},
        {0x1.11a3019a74826p+0, -0x1.10e45b3cae829p-4, -0x1.9b5ed72e6d974p-58},
        {0x1.107fbbe011080p+0, -0x1.ffa6911ab9309p-5, 0x1.cd9f1f95c2ef1p-59},
        {0x1.0f5edfab325a2p+0, -0x1.dda8adc67ee59p-5, 0x1.31936790bb3b2p-59},
        {0x1.0e40655826011p+0, -0x1.bbcebfc68f424p-5, 0x1.cd1862f854848p-59},
        {0x1.0d24456359e3ap+0, -0x1.9a187b573de81p-5, -0x1.b13b26f298a6ap-64},
        {0x1.0c0a7868b4171p+0, -0x1.788595a3577c8p-5, -0x1.2f7c4c5b3c8bdp-62},
        {0x1.0af2f722eecb5p+0, -0x1.5715c4c03cee1p-5, -0x1.5101dc4ebf91fp-59},
        {0x1.09ddba6af8360p+0, -0x1.35c8bfaa13069p-5, 0x1.50830a65543a8p-63},
        {0x1.08cabb37565e2p+0, -0x1.149e3e4005a8dp-5, 0x1.a9a4168fcebebp-60},
        {0x1.07b9f29b8eae2p+0, -0x1.e72bf2813ce6ap-6, 0x1.8a4bba6a354fap-60},
        {0x1.06ab59c7912fbp+0, -0x1.a55f548c5c427p-6, -0x1.f60d2fc36a0d9p-61},
        {0x1.059eea0727586p+0, -0x1.63d6178690bbep-6, 0x1.18ed4d357c9dcp-60},
        {0x1.04949cc1664c5p+0, -0x1.228fb1fea2e0ap-6, -0x1.3284991fe3d5cp-61},
        {0x1.038c6b78247fcp+0, -0x1.c317384c75f0dp-7, -0x1.806208c04c21fp-61},
        {0x1.02864fc7729e9p+0, -0x1.41929f968330cp-7, -0x1.3aae809b43dd0p-61},
        {0x1.0182436517a37p+0, -0x1.8121214586b02p-8, 0x1.c7d68c0d910f2p-62},
        {0x1.0000000000000p+0, 0x0.0p+0, 0x0.0p+0},
};

double oracle_plog(double u)
{
    /* (-1)^(k+1)/k, k = 2..7, each correctly rounded (pinned in tests). */
    static const double Q[6] = {
        -0x1.0000000000000p-1,  /* -1/2 */
        0x1.5555555555555p-2,   /* 1/3  */
        -0x1.0000000000000p-2,  /* -1/4 */
        0x1.999999999999ap-3,   /* 1/5  */
        -0x1.5555555555555p-3,  /* -1/6 */
        0x1.2492492492492p-3,   /* 1/7  */
    };
    const double LN2_HI = 0x1.62e42fee00000p-1;    /* ln 2, 32 significant bits */
    const double LN2_LO = 0x1.a39ef35793c76p-33;   /* fl(ln 2 - LN2_HI) */

    uint64_t b = double_to_bits(u);
    int e = (int)((b >> 52) & 0x7FF) - 1023;
    int i = (int)((b >> 45) & 0x7F);
    uint64_t mb = (b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
    if (i >= 53) {
        mb = mb - (1ull << 52);    /* m / 2, exact */
        e = e + 1;
    }
    double m = bits_to_double(mb);
    double r = fma(m, PLOG_TAB[i][0], -1.0);
    double q = Q[5];
    for (int k = 4; k >= 0; --k)
        q = fma(q, r, Q[k]);
    double r2 = r * r;
    double p = fma(r2, q, r);
    double ed = (double)e;
    double hi = fma(ed, LN2_HI, PLOG_TAB[i][1]);
    double lo = fma(ed, LN2_LO, PLOG_TAB[i][2]) + p;
    return hi + lo;
}

/* ------------------------------------------------------------------------ */
/* a3: propensities ("the more the reactants (and the rate) */
/* the highest the probability", e.g. I4 x pi; PAPER.md:93 state-dependent   */
/* infectivity).  a_j = k^_j * h_j with                                       */
/*   h_j = prod over reactant terms, in declared order, of C(x_s, m)         */
/*         (unordered combinations, R1), each product an fp64 op;  */
/*   k^_j = k_j, or max(0, k_j + d_j * x_mod) for a modified reaction (R4).  */
/* Returns OR_OK, or OR_ERR_NUMERIC with *bad = first non-finite reaction.   */
/* ------------------------------------------------------------------------ */
static double binom_factor(int64_t xs, int32_t m)
{
    double x = (double)xs;                   /* exact: counts < 2^53 */
    if (m == 1) return x;
    if (m == 2) return (x * (x - 1.0)) * 0.5;
    /* m == 3 */
    return ((x * (x - 1.0)) * (x - 2.0)) / 6.0;
}

int oracle_propensities(const oracle_model *M, const int64_t *x, double *a, int32_t *bad)
{
    for (int j = 0; j < M->R; ++j) {
        double h = 1.0;
        for (int q = 0; q < M->n_reac[j]; ++q) {
            double fct = binom_factor(x[M->reac_sp[3 * j + q]], M->reac_coef[3 * j + q]);
            h = (q == 0) ? fct : h * fct;
        }
        if (M->mass_action && !M->mass_action[j]) h = 1.0;   /* reactants only consume */
        double k = M->rate[j];
        if (M->mod_sp[j] >= 0) {
            double xm = (double)x[M->mod_sp[j]];
            k = k + M->mod_coef[j] * xm;     /* two roundings, no fma */
            if (k < 0.0) k = 0.0;            /* "0 <= beta_R5" */
        }
        a[j] = k * h;
        /* gates: a closed gate makes the propensity exactly 0 */
        int open = 1;
        for (int g = 0; M->n_gates && g < M->n_gates[j]; ++g) {
            int64_t xg = x[M->gate_sp[4 * j + g]];
            if (M->gate_kind[4 * j + g] == 0 ? !(xg > 0) : !(xg == 0)) open = 0;
        }
        if (!open) a[j] = 0.0;
        if (!isfinite(a[j])) {
            if (bad) *bad = j;
            return OR_ERR_NUMERIC;
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* a4 + a7: total propensity and selection, in one of two declared           */
/* summation orders (R13):                                         */
/*  mode 0 "sequential": c_j = c_{j-1} + a_j left to right, a0 = c_{R-1},    */
/*         j* = min{ j : c_j > r }.                                           */
/*  mode 1 "warp32" (mode 2 "warp16": the same with 16 lanes):              */
/*         P = ceil(R/32) contiguous reactions per lane l;                     */
/*         L_l = sequential sum of lane l's a_j;  Hillis-Steele inclusive     */
/*         scan over the 32 L_l with offsets 1,2,4,8,16 gives v_l; a0 = v_31; */
/*         lane* = min{ l : v_l > r };  p = v_{lane*-1} (0 for lane 0), then  */
/*         p += a_j over lane*'s reactions in order, j* = first j with p > r; */
/*         if none, j* = the largest j <= lane*'s last index with a_j > 0.    */
/*  mode 3 "warp16s" (the half-warp path since round 2): lane sums, scan and */
/*         lane* as mode 2; then lane*'s P propensities (padded with 0 to 16  */
/*         positions) are Hillis-Steele scanned over the 16 positions         */
/*         (offsets 1,2,4,8) into s_q, p_q = v_{lane*-1} + s_q (s_q for lane  */
/*         0), j* = lane*'s q-th reaction for the first q with p_q > r; if    */
/*         none, the fallback of mode 2.                                      */
/* r = u2 * a0 ("smallest j with sum_{i<=j} a_i > u2 a0").        */
/* ------------------------------------------------------------------------ */
static double total_sequential(const double *a, int R)
{
    double c = 0.0;
    for (int j = 0; j < R; ++j) c = c + a[j];
    return c;
}

static int select_sequential(const double *a, int R, double r)
{
    double c = 0.0;
    for (int j = 0; j < R; ++j) {
        c = c + a[j];
        if (c > r) return j;
    }
    return -1; /* unreachable when r < a0 (R12) */
}

/* The warp orders with L lanes (L = 32: mode 1 "warp32", L = 16: mode 2
 * "warp16", a half warp per trajectory): P = ceil(R/L) contiguous reactions
 * per lane, lane sums from 0.0 in order, inclusive Hillis-Steele scan over
 * the L lane sums with offsets 1, 2, 4, ... < L, a0 = v_{L-1}. */
static int mode_lanes(int mode) { return (mode == 2 || mode == 3) ? 16 : 32; }

static void warp_scan_mode(const double *a, int R, int L, int mode, double v[32])
{
    int P = (R + L - 1) / L;
    if (P < 1) P = 1;
    double lsum[32];
    for (int l = 0; l < L; ++l) {
        double s = 0.0;
        for (int j = l * P; j < (l + 1) * P && j < R; ++j) s = s + a[j];
        lsum[l] = s;
    }
    for (int l = 0; l < L; ++l) v[l] = lsum[l];
    for (int o = 1; o < L; o *= 2) {
        double nv[32];
        for (int l = 0; l < L; ++l) nv[l] = (l >= o) ? (v[l - o] + v[l]) : v[l];
        for (int l = 0; l < L; ++l) v[l] = nv[l];
    }
}

static int select_warp(const double *a, int R, int L, const double v[32], double r)
{
    int P = (R + L - 1) / L;
    if (P < 1) P = 1;
    int lane = -1;
    for (int l = 0; l < L; ++l) {
        if (v[l] > r) { lane = l; break; }
    }
    if (lane < 0) return -1;
    double p = (lane > 0) ? v[lane - 1] : 0.0;
    int last = (lane + 1) * P - 1;
    if (last > R - 1) last = R - 1;
    for (int j = lane * P; j <= last; ++j) {
        p = p + a[j];
        if (p > r) return j;
    }
    for (int j = last; j >= 0; --j)
        if (a[j] > 0.0) return j;
    return -1;
}

/* mode 3: the within-lane step as a 16-position Hillis-Steele scan (DESIGN.md
 * R13: the summation and selection order is declared per path; the paper is
 * silent). */
static int select_warp_scanned(const double *a, int R, const double v[32], double r)
{
    const int L = 16;
    int P = (R + L - 1) / L;
    if (P < 1) P = 1;
    int lane = -1;
    for (int l = 0; l < L; ++l) {
        if (v[l] > r) { lane = l; break; }
    }
    if (lane < 0) return -1;
    double s[16];
    for (int q = 0; q < 16; ++q) {
        const int j = lane * P + q;
        s[q] = (q < P && j < R) ? a[j] : 0.0;
    }
    for (int o = 1; o < 16; o *= 2) {
        double ns[16];
        for (int q = 0; q < 16; ++q) ns[q] = (q >= o) ? (s[q - o] + s[q]) : s[q];
        for (int q = 0; q < 16; ++q) s[q] = ns[q];
    }
    const double base = (lane > 0) ? v[lane - 1] : 0.0;
    int last = (lane + 1) * P - 1;
    if (last > R - 1) last = R - 1;
    for (int q = 0; q < P && lane * P + q <= last; ++q) {
        const double p = (lane > 0) ? base + s[q] : s[q];
        if (p > r) return lane * P + q;
    }
    for (int j = last; j >= 0; --j)
        if (a[j] > 0.0) return j;
    return -1;
}

/* Computes a0 and j* for given propensities and u2 (mode 0, 1, 2 or 3). */
int oracle_select(const double *a, int32_t R, int32_t mode, double u2, double *a0_out, int32_t *j_out)
{
    double a0, r;
    int j;
    if (mode == 0) {
        a0 = total_sequential(a, R);
        r = u2 * a0;
        j = (a0 > 0.0) ? select_sequential(a, R, r) : -1;
    } else {
        double v[32];
        const int L = mode_lanes(mode);
        warp_scan_mode(a, R, L, mode, v);
        a0 = v[L - 1];
        r = u2 * a0;
        j = (a0 > 0.0) ? (mode == 3 ? select_warp_scanned(a, R, v, r) : select_warp(a, R, L, v, r)) : -1;
    }
    *a0_out = a0;
    *j_out = j;
    return OR_OK;
}

/* One direct-method step with prescribed uniforms:
 * tau = -plog(u1) / a0; returns *j = -1 and tau = +inf when a0 == 0. */
int oracle_step(const oracle_model *M, const int64_t *x, double u1, double u2, int32_t mode,
                double *tau, int32_t *j)
{
    double *a = (double *)malloc(sizeof(double) * (M->R > 0 ? M->R : 1));
    int32_t bad = -1;
    int st = oracle_propensities(M, x, a, &bad);
    if (st != OR_OK) { free(a); *j = bad; return st; }
    double a0;
    oracle_select(a, M->R, mode, u2, &a0, j);
    if (a0 == 0.0) {
        *tau = INFINITY;
        *j = -1;
    } else {
        double E = -oracle_plog(u1);
        *tau = E / a0;
    }
    free(a);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* a6: grid alignment -- selective memory on a fixed grid (PAPER.md:143,     */
/* :147 "aligns simulation points ... according to simulation time";         */
/* DESIGN.md R14, R15).  Grid s_k = k * dt, k = 0..K, K = floor(t_end/dt +   */
/* 1e-9).  The state held at s_k is the state just before the first event    */
/* with time > s_k (an event exactly at s_k is included: right-continuous    */
/* zero-order hold).                                                          */
/* ------------------------------------------------------------------------ */
int64_t oracle_grid_K(double t_end, double dt)
{
    return (int64_t)floor(t_end / dt + 1e-9);
}

typedef struct {
    int32_t S;
    int64_t K;
    double dt;
    int64_t k;            /* next grid index to emit */
    int32_t *grid_x;      /* [G*S] or NULL */
    uint64_t *grid_e;     /* [G] or NULL */
    double *grid_t;       /* [G] or NULL */
    uint64_t near_ties;
    int32_t overflow;
} grid_cursor;

/* Emit every grid point s_k with s_k < tn (tn = candidate event time, or
 * +inf for an absorbing state).  x = held state, t = time of the last
 * applied event (meaningful if e > 0). */
static void grid_emit_before(grid_cursor *g, const int64_t *x, double t, uint64_t e, double tn)
{
    while (g->k <= g->K) {
        double sk = (double)g->k * g->dt;
        if (!(tn > sk)) break;
        double tol = 1e-9 * sk;
        int near = 0;
        if (isfinite(tn) && fabs(tn - sk) <= tol) near = 1;
        if (e > 0 && fabs(t - sk) <= tol) near = 1;
        g->near_ties += (uint64_t)near;
        if (g->grid_x) {
            for (int s = 0; s < g->S; ++s) {
                if (x[s] > 2147483647LL) g->overflow = 1;
                g->grid_x[g->k * g->S + s] = (int32_t)x[s];
            }
        } else {
            for (int s = 0; s < g->S; ++s)
                if (x[s] > 2147483647LL) g->overflow = 1;
        }
        if (g->grid_e) g->grid_e[g->k] = e;
        if (g->grid_t) g->grid_t[g->k] = (e > 0) ? t : 0.0;
        g->k += 1;
    }
}

/* Test hook for the aligner alone: feed a prescribed event stream
 * (times[i], state after event i) and the initial state; the stream ends at
 * the first event with time > s_K, or, if exhausted, is held to the end. */
int oracle_align_events(int32_t S, const int64_t *x0, int64_t n_events, const double *times,
                        const int64_t *states, double t_end, double dt, int32_t *grid_x,
                        uint64_t *grid_e, double *grid_t, uint64_t *near_ties)
{
    grid_cursor g = {S, oracle_grid_K(t_end, dt), dt, 0, grid_x, grid_e, grid_t, 0, 0};
    const int64_t *x = x0;
    double t = 0.0;
    uint64_t e = 0;
    for (int64_t i = 0; i < n_events && g.k <= g.K; ++i) {
        grid_emit_before(&g, x, t, e, times[i]);
        if (g.k > g.K) break;
        x = states + i * S;
        t = times[i];
        e += 1;
    }
    grid_emit_before(&g, x, t, e, INFINITY);
    if (near_ties) *near_ties = g.near_ties;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* a1-a8: one trajectory ("Given the current state of the        */
/* system, a single transition amongst the possible ones is selected, and    */
/* the state updated accordingly. The Gillespie's algorithm [8] determines   */
/* the next transition and the time at which it occurs").                    */
/* ------------------------------------------------------------------------ */
#define FNV_OFFSET 0xcbf29ce484222325ull
#define FNV_PRIME 0x100000001b3ull

/* As oracle_trajectory, also recording the applied events in order: their
 * times ev_t[i] and reactions ev_j[i] for i < ev_cap (either may be NULL);
 * *ev_n receives the number of applied events.  This is the full event
 * stream of the trajectory ("the full simulation results"),
 * used by the union-time selective memory (NEXT 2). */
int oracle_trajectory_events(const oracle_model *M, uint64_t id, uint64_t seed, double t_end, double dt,
                             int32_t mode, int32_t *grid_x, uint64_t *grid_e, double *grid_t,
                             oracle_summary *sum, int64_t ev_cap, double *ev_t, int32_t *ev_j, int64_t *ev_n);

int oracle_trajectory(const oracle_model *M, uint64_t id, uint64_t seed, double t_end, double dt,
                      int32_t mode, int32_t *grid_x, uint64_t *grid_e, double *grid_t,
                      oracle_summary *sum)
{
    return oracle_trajectory_events(M, id, seed, t_end, dt, mode, grid_x, grid_e, grid_t, sum, 0, NULL, NULL, NULL);
}

int oracle_trajectory_events(const oracle_model *M, uint64_t id, uint64_t seed, double t_end, double dt,
                             int32_t mode, int32_t *grid_x, uint64_t *grid_e, double *grid_t,
                             oracle_summary *sum, int64_t ev_cap, double *ev_t, int32_t *ev_j, int64_t *ev_n)
{
    int S = M->S, R = M->R;
    int64_t *x = (int64_t *)malloc(sizeof(int64_t) * (S > 0 ? S : 1));
    double *a = (double *)malloc(sizeof(double) * (R > 0 ? R : 1));
    for (int s = 0; s < S; ++s) x[s] = M->x0[s];

    grid_cursor g = {S, oracle_grid_K(t_end, dt), dt, 0, grid_x, grid_e, grid_t, 0, 0};
    double t = 0.0;
    uint64_t e = 0;
    uint64_t hash = FNV_OFFSET;
    int32_t absorbed = 0, status = OR_OK, bad = -1;
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};

    for (;;) {
        /* a2: one Philox block per candidate event */
        uint32_t ctr[4] = {(uint32_t)e, (uint32_t)(e >> 32), (uint32_t)id, (uint32_t)(id >> 32)};
        uint32_t o[4];
        oracle_philox4x32_10(ctr, key, o);
        double u1 = oracle_u53(((uint64_t)o[1] << 32) | o[0]);
        double u2 = oracle_u53(((uint64_t)o[3] << 32) | o[2]);

        /* a3 */
        status = oracle_propensities(M, x, a, &bad);
        if (status != OR_OK) break;

        /* a4 */
        double a0, v[32];
        if (mode == 0) {
            a0 = total_sequential(a, R);
        } else {
            warp_scan_mode(a, R, mode_lanes(mode), mode, v);
            a0 = v[mode_lanes(mode) - 1];
        }

        /* a5 */
        if (a0 == 0.0) {
            grid_emit_before(&g, x, t, e, INFINITY);
            absorbed = 1;
            break;
        }
        if (!isfinite(a0)) { status = OR_ERR_NUMERIC; bad = -1; break; }
        double E = -oracle_plog(u1);
        double tau = E / a0;
        double tn = t + tau;

        /* a6 */
        grid_emit_before(&g, x, t, e, tn);
        if (g.k > g.K) break;

        /* a7 */
        double r = u2 * a0;
        int j = (mode == 0) ? select_sequential(a, R, r)
              : (mode == 3) ? select_warp_scanned(a, R, v, r) : select_warp(a, R, mode_lanes(mode), v, r);

        /* a8 */
        for (int s = 0; s < S; ++s) x[s] += M->nu[(int64_t)j * S + s];
        t = tn;
        if ((int64_t)e < ev_cap) {
            if (ev_t) ev_t[e] = tn;
            if (ev_j) ev_j[e] = j;
        }
        e += 1;
        hash = (hash ^ (uint64_t)j) * FNV_PRIME;
    }
    if (status == OR_OK && g.overflow) status = OR_ERR_OVERFLOW;
    if (ev_n) *ev_n = (int64_t)e;
    if (sum) {
        sum->events = e;
        sum->hash = hash;
        sum->t_last = t;
        sum->near_ties = g.near_ties;
        sum->absorbed = absorbed;
        sum->status = status;
        sum->err_reaction = bad;
        sum->pad = 0;
    }
    free(x);
    free(a);
    return status;
}

/* ------------------------------------------------------------------------ */
/* a9-a10 (oracle form, R19): exact integer moments               */
/* S1 = sum x, S2 = sum x^2 (128-bit) per (k, s) over the trajectories, then */
/* mean = S1 / n and population variance = (n S2 - S1^2) / n^2 (*/
/* DESIGN.md R18), each rounded once to double from an exact numerator.      */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t n;
    int64_t cells;       /* G*S */
    int64_t *s1;         /* [cells] */
    __int128 *s2;        /* [cells] */
} moment_acc;

static void acc_add(moment_acc *A, const int32_t *sample)
{
    for (int64_t c = 0; c < A->cells; ++c) {
        int64_t v = sample[c];
        A->s1[c] += v;
        A->s2[c] += (__int128)v * v;
    }
    A->n += 1;
}

static void acc_finalize(const moment_acc *A, double *mean, double *var)
{
    for (int64_t c = 0; c < A->cells; ++c) {
        if (A->n == 0) { mean[c] = 0.0; var[c] = 0.0; continue; }
        __int128 n = A->n;
        __int128 num = n * A->s2[c] - (__int128)A->s1[c] * A->s1[c];
        long double nl = (long double)A->n;
        mean[c] = (double)((long double)A->s1[c] / nl);
        var[c] = (double)((long double)num / (nl * nl));
    }
}

/* Exact moments of n given samples (row-major [n][cells]). */
int oracle_moments(int64_t n, int64_t cells, const int32_t *samples, double *mean, double *var)
{
    moment_acc A = {0, cells, calloc((size_t)cells, sizeof(int64_t)),
                    calloc((size_t)cells, sizeof(__int128))};
    for (int64_t i = 0; i < n; ++i) acc_add(&A, samples + i * cells);
    acc_finalize(&A, mean, var);
    free(A.s1);
    free(A.s2);
    return OR_OK;
}

/* Whole ensemble over an explicit id list: trajectories in the given order,
 * exact moments, optional per-trajectory outputs (each may be NULL):
 *   grid_x [n_ids][G][S], grid_e [n_ids][G], grid_t [n_ids][G], sums [n_ids].
 * Returns the first non-OK trajectory status (all trajectories still run). */
int oracle_run(const oracle_model *M, int64_t n_ids, const uint64_t *ids, uint64_t seed,
               double t_end, double dt, int32_t mode, double *mean, double *var,
               int32_t *grid_x, uint64_t *grid_e, double *grid_t, oracle_summary *sums)
{
    int64_t G = oracle_grid_K(t_end, dt) + 1;
    int64_t cells = G * M->S;
    moment_acc A = {0, cells, calloc((size_t)(cells ? cells : 1), sizeof(int64_t)),
                    calloc((size_t)(cells ? cells : 1), sizeof(__int128))};
    int32_t *gx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cells ? cells : 1));
    int first = OR_OK;
    for (int64_t i = 0; i < n_ids; ++i) {
        oracle_summary s;
        int st = oracle_trajectory(M, ids[i], seed, t_end, dt, mode, gx,
                                   grid_e ? grid_e + i * G : NULL,
                                   grid_t ? grid_t + i * G : NULL, &s);
        if (st != OR_OK && first == OR_OK) first = st;
        acc_add(&A, gx);
        if (grid_x) memcpy(grid_x + i * cells, gx, sizeof(int32_t) * (size_t)cells);
        if (sums) sums[i] = s;
    }
    if (mean && var) acc_finalize(&A, mean, var);
    free(gx);
    free(A.s1);
    free(A.s2);
    return first;
}

/* Array conveniences for the pin tests (plain loops over the scalar forms). */
void oracle_plog_n(int64_t n, const double *u, double *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_plog(u[i]);
}

void oracle_philox_n(int64_t n, const uint32_t *ctr, const uint32_t key[2], uint32_t *out)
{
    for (int64_t i = 0; i < n; ++i) oracle_philox4x32_10(ctr + 4 * i, key, out + 4 * i);
}

void oracle_u53_n(int64_t n, const uint64_t *w, double *out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = oracle_u53(w[i]);
}

int oracle_abi_version(void) { return 1; }
