// Host model of the count kernel's D2 walk over one config-5 SCC (tools/ note, DESIGN 6.7): passes per
// extension when a pass makes P pops before its take (P = 0: one move per pass).  Input: /tmp/sim/scc.txt,
// the in-SCC successor lists of config 5's first SCC (one line per local vertex).
// gcc -O2 -o /tmp/m tools/d2_pass_model.c && /tmp/m 8
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
int n=56, sc[64][2], ns[64];
int main(int argc,char**argv){
  FILE*f=fopen("/tmp/sim/scc.txt","r"); char line[256];
  for(int v=0;v<n;v++){if(!fgets(line,256,f))return 1; ns[v]=sscanf(line,"%d %d",&sc[v][0],&sc[v][1]);}
  int nst=argc>1?atoi(argv[1]):8;
  for(int P=0;P<=4;P++){
  long long takes=0,passes=0;
  for(int s=0;s<nst;s++){
    uint64_t M=1ull<<s; int l=0; uint8_t path[70]; int pend[70]; path[0]=s;
    int cur[2], nc=0;
    for(int i=0;i<ns[s];i++){int t=sc[s][i]; if(t==s||!((M>>t)&1)) cur[nc++]=t;}
    int done=0;
    while(!done){
      passes++;
      int npop = P==0 ? 1 : P;   // P=0: unified (pop OR take)
      int popped=0;
      for(int k=0;k<npop;k++){
        if(nc==0){ if(l==0){done=1;break;} M&=~(1ull<<path[l]); l--; nc=0; if(pend[l]!=0xff){cur[0]=pend[l];nc=1;} popped=1; }
      }
      if(done) break;
      if(P==0 && popped) continue;
      if(nc==0) continue;
      int w=cur[0]; int rest=(nc==2)?cur[1]:0xff; takes++;
      if(w==s){ if(rest!=0xff){cur[0]=rest;nc=1;} else nc=0; continue;}
      uint64_t Mw=M|(1ull<<w); int cw[2],ncw=0;
      for(int i=0;i<ns[w];i++){int t=sc[w][i]; if(t==s||!((Mw>>t)&1)) cw[ncw++]=t;}
      if(ncw==0){ if(rest!=0xff){cur[0]=rest;nc=1;} else nc=0; continue;}
      pend[l]=rest; l++; path[l]=w; M=Mw; cur[0]=cw[0]; cur[1]=ncw>1?cw[1]:0; nc=ncw;
    }
  }
  printf("P=%d passes/take %.3f\n",P,(double)passes/takes);
  }
}
