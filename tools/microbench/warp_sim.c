// warp_sim.c — warp-lockstep CPU simulation of the product DFS step (not product code).
// Replays the always-descend kernel (nq_kernel.cuh) for 32 lanes in lockstep over the
// folded frontier (expensive end first) and counts, per warp-step, the lanes that push
// and pop and the shared-memory wavefronts of the V4 stack under two cost models:
//   max-group: max over the 8 bank groups (t mod 8) of active lanes;
//   quarter:   one wavefront per quarter-warp (lanes 8q..8q+7) with an active lane.
// gcc -O2 -o warp_sim warp_sim.c && ./warp_sim 18 6 16     (N, R, record stride)
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
typedef struct { uint32_t C,l,r,a; } F;
typedef struct { uint32_t cols, diag, anti, row; } Sub;
static Sub* subs; static size_t nsubs;
static int N; static uint32_t MASK;
static void gen(uint32_t c,uint32_t d,uint32_t a,int row,int R,int mult, size_t* cap){
  if(row==R){ if(nsubs==*cap){*cap*=2; subs=realloc(subs,*cap*sizeof(Sub));} subs[nsubs++] = (Sub){c,d,a,R|(mult<<8)}; return;}
  uint32_t v = MASK & ~(c|d|a);
  while(v){uint32_t p=v&-v; v^=p; gen(c|p,(d|p)<<1,(a|p)>>1,row+1,R,mult,cap);}
}
int main(int argc,char**argv){
  N=atoi(argv[1]); int R=atoi(argv[2]); int stride = argc>3?atoi(argv[3]):1;
  MASK=(1u<<N)-1; size_t cap=1<<20; subs=malloc(cap*sizeof(Sub));
  for(int c=0;c<N/2;c++){uint32_t p=1u<<c; gen(p,p<<1,p>>1,1,R,2,&cap);}
  if(N&1){int c=(N-1)/2; uint32_t p=1u<<c; uint32_t lh=(1u<<(c-1))-1; uint32_t v=(MASK&~(p|p<<1|p>>1))&lh;
    while(v){uint32_t q=v&-v; v^=q; gen(p|q,((p<<1)|q)<<1,((p>>1)|q)>>1,2,R,2,&cap);} }
  // reverse order (expensive first), take every stride-th
  size_t next = 0; 
  F stk[32][32]; int sp[32]; F cur[32]; int busy[32];
  for(int t=0;t<32;t++){busy[t]=0;sp[t]=0;cur[t]=(F){0,0,0,0};}
  uint64_t steps=0, busysteps=0, pushes=0, pops=0, stay=0, wst=0, wld=0, idealst=0, idealld=0, nodes=0;
  uint64_t wqst=0,wqld=0; uint64_t hist_push[33]={0}, hist_pop[33]={0};
  uint64_t costdist_st[9]={0};
  int done=0; uint64_t iter=0;
  while(1){
    // refill idle lanes
    int any=0;
    for(int t=0;t<32;t++){
      if(cur[t].a==0){ busy[t]=0;
        while(next*stride < nsubs){ Sub s=subs[nsubs-1-next*stride]; next++;
          uint32_t C=MASK&~s.cols; uint32_t a=C&~(s.diag|s.anti);
          if(a){cur[t]=(F){C,s.diag,s.anti,a}; sp[t]=0; busy[t]=1; break;} }
      }
      if(cur[t].a) any=1;
    }
    if(!any) break;
    for(int k=0;k<32;k++){
      int gp[8]={0}, gl[8]={0}; int np=0, nl=0; int qpush[32]={0}, qpop[32]={0};
      for(int t=0;t<32;t++){
        F f=cur[t]; if(!f.a) continue; 
        nodes++;
        uint32_t p=f.a&-f.a; f.a^=p; int pushed=0;
        if(f.a){ stk[t][sp[t]++]=f; gp[t&7]++; np++; pushed=1; qpush[t]=1;}
        uint32_t C=f.C-p, l=(f.l+p)<<1, r=(f.r+p)>>1; uint32_t a=C&~(l|r);
        if(a==0){ // pop
          if(sp[t]>0){ if(pushed) stay++; cur[t]=stk[t][--sp[t]]; gl[t&7]++; nl++; qpop[t]=1; }
          else { cur[t]=(F){0,0,0,0}; }
        } else cur[t]=(F){C,l,r,a};
      }
      int mst=0,mld=0; for(int g=0;g<8;g++){ if(gp[g]>mst)mst=gp[g]; if(gl[g]>mld)mld=gl[g]; }
      { int qs=0,ql=0; for(int q=0;q<4;q++){ int a1=0,a2=0; for(int t=8*q;t<8*q+8;t++){ a1|=qpush[t]; a2|=qpop[t]; } qs+=a1; ql+=a2; } wqst+=qs; wqld+=ql; }
      wst+=mst; wld+=mld; idealst += (np*16+127)/128; idealld += (nl*16+127)/128;
      pushes+=np; pops+=nl; hist_push[np]++; hist_pop[nl]++; costdist_st[mst]++;
      steps++;
    }
  }
  printf("N=%d R=%d stride=%d subs=%zu nodes=%llu warp-steps=%llu\n",N,R,stride,nsubs,(unsigned long long)nodes,(unsigned long long)steps);
  printf("push/node %.4f pop/node %.4f stay/push %.4f\n",(double)pushes/nodes,(double)pops/nodes,(double)stay/pushes);
  printf("lanes busy/step %.2f  STS wf/step %.3f (ideal %.3f)  LDS wf/step %.3f (ideal %.3f)  wf/node %.4f ideal %.4f\n",
     (double)nodes/steps,(double)wst/steps,(double)idealst/steps,(double)wld/steps,(double)idealld/steps,(double)(wst+wld)/nodes,(double)(idealst+idealld)/nodes);
  printf("quarter model: STS %.3f LDS %.3f per step, wf/node %.4f\n",(double)wqst/steps,(double)wqld/steps,(double)(wqst+wqld)/nodes);
  printf("mean pushers/step %.2f popper/step %.2f\n",(double)pushes/steps,(double)pops/steps);
  printf("STS cost dist:"); for(int i=0;i<=4;i++) printf(" %d:%.3f",i,(double)costdist_st[i]/steps); printf("\n");
  return 0;
}
