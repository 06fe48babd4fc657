"""Copy nlohmann/json 3.11.3 and revert cudnn-frontend's compact-array patch.

TEST INFRASTRUCTURE ONLY (used by oracle/Makefile to build oracle/_ref).
The venv's json.hpp prints integer arrays on one line ("Custom from FE");
stock nlohmann prints one element per line, which the reference's byte-stable
fixture tests/fixtures/fig6_plan.json expects.  Only JSON text changes.
"""
import sys

src, dst = sys.argv[1], sys.argv[2]
text = open(src, encoding="utf-8").read()
patched = (
    "                if (pretty_print && (elementType != value_t::number_integer) &&\n"
    "                    (elementType != value_t::number_unsigned))\n"
)
stock = "                if (pretty_print)\n"
if patched in text:
    text = text.replace(patched, stock, 1)
open(dst, "w", encoding="utf-8").write(text)
