# usage: bash scripts/gpu_all.sh <tag> [pytest -k expr]   (smoke, GPU tests, bench, ncu of the scan)
TAG=${1:-run}
bash scripts/gpu_check.sh "$TAG" "$2"
bash scripts/gpu_prof.sh "$TAG"
