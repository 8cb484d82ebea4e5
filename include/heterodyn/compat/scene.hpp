// Reference include name (/root/reference/proj/src/scene.hpp) for drop-in callers:
// compile with -I include/heterodyn/compat.  Everything is declared in ../solver.hpp.
#pragma once
#include "../solver.hpp"
