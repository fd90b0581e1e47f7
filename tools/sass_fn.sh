# Usage: bash tools/sass_fn.sh LIB.so PATTERN  -- SASS of the first function whose name matches PATTERN
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{f = ($0 ~ pat) && !seen; if (f) seen = 1} f'
