mkdir -p gpurun_out/s3o
V="MODE=2,COPY=1;MODE=2,COPY=2,WS=0;MODE=2,COPY=2,WS=1"
for code in 20,40,gf64,1 40,20,gf64 30,30,gf64,0 12,48,gf64,1 8,4,gf16; do
  timeout 900 python tools/tune.py --code $code --frag 9600000 --steps 10 --rounds 3 --variants "$V" > gpurun_out/s3o/k_${code//,/_}.jsonl 2>&1
done
