# A/B of programmatic dependent launch: off / early trigger / implicit trigger
run() {  # label workload steps env...
  local label=$1 w=$2 n=$3; shift 3
  env "$@" python bench.py --workload $w --no-baselines --no-sweep --steps $n --warmup 5 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $label', round(d['value']), round(d['ms_per_step'],4))"
}
NT=paper_2410_22254_b200/_lib_nt/libtlk.so
for rep in 1 2; do
for w in cnn mlp; do
  run off $w 200 TLK_PDL=0; run trig $w 200 TLK_PDL=1; run notrig $w 200 TLK_LIB=$NT
done; done
for w in resnet18 xformer gpt; do
  run off $w 20 TLK_PDL=0; run trig $w 20 TLK_PDL=1; run notrig $w 20 TLK_LIB=$NT
done
