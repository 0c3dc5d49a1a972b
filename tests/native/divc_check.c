/* Exhaustive-style check of the update kernels' division by the per-step bias
 * correction (device.cuh divc, R21): for b = fl32(1 - beta^t),
 * beta in {0.9, 0.999}, y = RN(1/b), q = RN(a y), r = fma(-q, b, a),
 * q' = fma(r, y, q) must equal the IEEE quotient a / b bit for bit for every a
 * with |a| >= 2^-100 (Markstein's theorem; smaller |a| take the IEEE division
 * in the kernel).  argv[1] = cases per divisor.  Exit code = mismatches (0 ok). */
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
static uint64_t s=88172645463325252ull;
static uint64_t xr(){ s^=s<<13; s^=s>>7; s^=s<<17; return s; }
int main(int argc, char** argv){
  const int per = argc > 1 ? atoi(argv[1]) : 20000;
  double betas[2]={0.9,0.999};
  long long bad=0, tot=0;
  for(int bi=0;bi<2;bi++){
    float beta=(float)betas[bi];
    for(int t=1;t<=200000;t+= (t<2000?1:37)){
      float b=(float)(1.0-pow((double)beta,(double)t));
      float y=(float)(1.0/(double)b);   /* RN(1/b): double then round is correct here (no double rounding issue? check) */
      /* correctly rounded reciprocal via fp32 division */
      float y2 = 1.0f / b;
      if (y != y2) { printf("recip mismatch t=%d\n", t); }
      for(int it=0; it<per; it++){
        uint32_t u=(uint32_t)xr();
        /* random exponent in [2^-100, 2^60] range, random mantissa, random sign */
        uint32_t e = 27 + (xr() % 160);
        u = (u & 0x807FFFFFu) | (e << 23);
        float a; memcpy(&a,&u,4);
        float q = a*y;
        float r = fmaf(-q, b, a);
        float q1 = fmaf(r, y, q);
        float ref = a / b;
        tot++;
        if (memcmp(&q1,&ref,4)) { bad++; if (bad<10) printf("bad t=%d a=%a b=%a q1=%a ref=%a\n",t,a,b,q1,ref); }
      }
    }
  }
  printf("tot %lld bad %lld\n", tot, bad);
  return bad ? 1 : 0;
}
