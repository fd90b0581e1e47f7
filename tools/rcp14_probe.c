/* Probe of vrcp14pd followed by vrndscalepd(0x58) -- the reciprocal step of
 * Intel SVML __svml_log8_ha -- on the AVX-512 host: prints the 16 mantissa
 * thresholds at which the rounded reciprocal changes (restated as kSvLogTh in
 * paper_2605_08699_b200/csrc/libm_restated.cuh and SVLOG_TH in oracle.c)
 * and checks monotonicity on 2e8 random mantissas.
 *     gcc -O2 -mavx512f -o rcp14_probe tools/rcp14_probe.c && ./rcp14_probe */
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>
static double rr(double m){ __m128d v=_mm_set_sd(m); __m128d r=_mm_rcp14_sd(v,v); r=_mm_roundscale_sd(r,r,0x58); return _mm_cvtsd_f64(r);}
static uint64_t db(double d){uint64_t u; memcpy(&u,&d,8); return u;}
static double bd(uint64_t u){double d; memcpy(&d,&u,8); return d;}
int main(){
  double th[40]; int nt=0;
  /* scan boundaries: rr is nonincreasing in m on [1,2) */
  uint64_t lo_b=db(1.0), hi_b=db(2.0)-1;
  double cur = rr(1.0);
  uint64_t a = lo_b;
  while (1) {
    /* find first m > a with rr(m) != cur, by exponential+binary search over bit patterns */
    uint64_t lo=a, hi=hi_b;
    if (rr(bd(hi))==cur) break;
    while (hi-lo>1){ uint64_t mid=lo+(hi-lo)/2; if (rr(bd(mid))==cur) lo=mid; else hi=mid; }
    th[nt++]=bd(hi); printf("rr=%a until m<%a (%.17g) then %a\n", cur, bd(hi), bd(hi), rr(bd(hi)));
    cur = rr(bd(hi)); a=hi;
  }
  /* verify: random m */
  uint64_t s=88172645463325252ull; long bad=0;
  for (long i=0;i<200000000;i++){ s^=s<<13; s^=s>>7; s^=s<<17; double m=bd(db(1.0) | (s & 0xfffffffffffffull));
    int k=0; while(k<nt && m>=th[k]) k++; double pred = (k==0)? rr(1.0) : rr(th[k-1]);
    if (pred != rr(m)) { bad++; if (bad<5) printf("nonmono m=%a\n", m);} }
  printf("nt=%d bad=%ld\n", nt, bad);
}
