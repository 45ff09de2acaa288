# GPU-side latency of one loopback all-reduce vs size, CUDA-graph replay (no host launch cost).
S=1024,4096,16384,65536,262144,1048576,4194304
for d in 8 2x4 2x2x2; do
python scripts/lb_microbench.py --graph --dims $d --sizes $S --algo 1 | sed "s/^/hier,/"
python scripts/lb_microbench.py --graph --dims $d --sizes 1024,4096,16384,65536,262144,1048576 --algo 2 --oneshot-max 1000000000 | sed "s/^/oneshot,/"
done
python scripts/lb_microbench.py --graph --P 2 --dims 2 --sizes $S --algo 1 | sed "s/^/hier,/"
python scripts/lb_microbench.py --graph --P 2 --dims 2 --sizes 1024,65536,262144,1048576 --algo 2 --oneshot-max 1000000000 | sed "s/^/oneshot,/"
python scripts/lb_microbench.py --graph --P 4 --dims 2x2 --sizes $S --algo 1 | sed "s/^/hier,/"
python scripts/lb_microbench.py --graph --P 4 --dims 2x2 --sizes 1024,65536,262144,1048576 --algo 2 --oneshot-max 1000000000 | sed "s/^/oneshot,/"
