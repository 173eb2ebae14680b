// Developer study (not product code): per-level duplication of BFS successors in the token ring
// (generated vs distinct per level / per frontier chunk).  gcc -O2 -o dedup_study dedup_study.c; ./dedup_study N CHUNKS
// token ring BFS duplication study: per level, successors generated vs distinct (whole level, and per chunk)
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
static int N;
static uint64_t mix(uint64_t z){z=(z^(z>>30))*0xBF58476D1CE4E5B9ull;z=(z^(z>>27))*0x94D049BB133111EBull;return z^(z>>31);}
typedef struct {uint64_t *k; uint64_t cap, n;} set;
static int ins(set*s, uint64_t key){ key+=1; uint64_t i=mix(key)&(s->cap-1); while(s->k[i]){ if(s->k[i]==key) return 0; i=(i+1)&(s->cap-1);} s->k[i]=key; s->n++; return 1;}
static void clr(set*s){memset(s->k,0,s->cap*8); s->n=0;}
static int get(uint64_t s,int i){return (s>>(3*i))&7;}
static uint64_t put(uint64_t s,int i,int v){return (s&~(7ull<<(3*i)))|((uint64_t)v<<(3*i));}
static int succ(uint64_t s, uint64_t*out){int n=0; for(int i=0;i<N;i++){int x=get(s,i);
  if(x==0) out[n++]=put(s,i,1); else if(x==2) out[n++]=put(s,i,3); else if(x==3) out[n++]=put(s,i,4);
  else if(x==1){int j=(i+1)%N; if(get(s,j)==4){uint64_t t=put(s,i,2); t=put(t,j,0); out[n++]=t;}}}
  return n;}
int main(int argc,char**argv){N=atoi(argv[1]); int chunks=argc>2?atoi(argv[2]):1;
  uint64_t total=2ull*N; for(int i=1;i<N;i++) total*=3;
  set vis={calloc(1ull<<34>>((N<15)?8:4),8),(1ull<<34)>>((N<15)?8:4),0};
  uint64_t lcap=1; while(lcap<total) lcap<<=1; lcap<<=1;
  set lv={calloc(lcap,8),lcap,0};
  uint64_t *F=malloc(total*8),*Fn=malloc(total*8); uint64_t nF=1; uint64_t s0=0; for(int i=1;i<N;i++) s0=put(s0,i,2); F[0]=s0; ins(&vis,s0);
  uint64_t G=0,D=0,DC=0,S=1; int level=0; uint64_t out[64];
  while(nF){ uint64_t nn=0,g=0,dc=0; clr(&lv);
    for(int c=0;c<chunks;c++){ set cs=lv; // per-chunk distinct counted by clearing a second set
      uint64_t lo=nF*c/chunks, hi=nF*(c+1)/chunks; static set ch={0}; if(!ch.k){ch.cap=lcap; ch.k=calloc(lcap,8);} clr(&ch);
      for(uint64_t i=lo;i<hi;i++){int n=succ(F[i],out); g+=n; for(int k=0;k<n;k++){ ins(&lv,out[k]); dc+=ins(&ch,out[k]); if(ins(&vis,out[k])) Fn[nn++]=out[k];}}
    }
    G+=g; D+=lv.n; DC+=dc; S+=nn;
    if(level%10==0) fprintf(stderr,"L%d front %lu gen %lu distinct %lu chunkdistinct %lu new %lu\n",level,nF,g,lv.n,dc,nn);
    uint64_t*t=F;F=Fn;Fn=t;nF=nn;level++;}
  printf("N=%d chunks=%d states=%lu levels=%d generated=%lu distinct_per_level=%lu (%.2fx) distinct_per_chunk=%lu (%.2fx)\n",N,chunks,S,level,G,D,(double)G/D,DC,(double)G/DC);
}
