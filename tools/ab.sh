# A/B helper: ab.sh <tag> <env...> : config-5 bench line without the slow legs
tag=$1; shift
env "$@" python bench.py --no-cpu-baseline --no-e2e --no-solve > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
